# Launch list of one bench step + full captures of the top kernels. Run under gpurun (1 GPU).
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-extras > gpurun_out/bench_ncu.json 2>&1; echo "launches rc=$?"
M=$((1<<20))
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/gemm_qkv python tools/gemm_once.py $M 2304 768 7 > /dev/null 2>&1; echo "gemm_qkv rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/gemm_out python tools/gemm_once.py $M 768 768 2 > /dev/null 2>&1; echo "gemm_out rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/gemm_fc1 python tools/gemm_once.py $M 3072 768 1 > /dev/null 2>&1; echo "gemm_fc1 rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/gemm_fc2 python tools/gemm_once.py $M 768 3072 2 > /dev/null 2>&1; echo "gemm_fc2 rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attention -s 1 -c 1 -o gpurun_out/attn python tools/attn_once.py 2048 512 > /dev/null 2>&1; echo "attn rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:layernorm -s 1 -c 1 -o gpurun_out/ln python bench.py --steps 1 --warmup 0 --no-extras --batch 2048 > /dev/null 2>&1; echo "ln rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:ms_merge_pass -s 3 -c 1 -o gpurun_out/tau_merge python tools/tau_once.py > /dev/null 2>&1; echo "tau rc=$?"
ls -la gpurun_out

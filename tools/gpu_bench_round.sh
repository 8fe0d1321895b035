# Round bench + evidence capture (run under gpurun). Never multi-rank under ncu.
set -x
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# per-launch device times of one step (cold-cache, serialised: compare shares)
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-extras > gpurun_out/bench_ncu.json 2>&1
# full capture of the dominant kernel (tcgen05 GEMM, FC1 shape) and of attention
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/gemm_fc1_full python tools/gemm_once.py 1048576 3072 768 1 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/gemm_out_full python tools/gemm_once.py 1048576 768 768 2 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:ms_merge_pass -s 3 -c 1 -o gpurun_out/tau_merge_full python tools/tau_once.py > /dev/null 2>&1
ls -la gpurun_out
cat gpurun_out/bench.json gpurun_out/bench_ref.json

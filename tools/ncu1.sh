set -x
mkdir -p gpurun_out
M=$((1<<20))
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/gemm2sm_fc1 python tools/gemm_once.py $M 3072 768 1 > gpurun_out/ncu_gemm2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_kernel -s 1 -c 1 -o gpurun_out/gemm1sm_fc1 python tools/gemm_once.py $((M+128)) 3072 768 1 > gpurun_out/ncu_gemm1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attention -s 1 -c 1 -o gpurun_out/attn python tools/attn_once.py 2048 512 > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out

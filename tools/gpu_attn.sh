mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_ranker.py tests/test_gpu_attention_bwd.py tests/test_gpu_gemm.py -q -p no:cacheprovider --timeout 120 --timeout-method thread -rf -x > gpurun_out/attn_tests.log 2>&1
grep -v "^  File\|^    " gpurun_out/attn_tests.log | grep -v "^$" | tail -25
timeout -s KILL 120 python tools/probe_attn.py > gpurun_out/probe_attn.log 2>&1; cat gpurun_out/probe_attn.log
timeout -s KILL 120 python tools/probe_gemm.py > gpurun_out/probe_gemm.log 2>&1; cat gpurun_out/probe_gemm.log
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attention_fwd -s 1 -c 1 -o gpurun_out/attn3 python tools/attn_once.py 2048 512 > /dev/null 2>&1; echo "ncu rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/gemm_out2 python tools/gemm_once.py 1048576 768 768 2 > /dev/null 2>&1; echo "ncu rc=$?"

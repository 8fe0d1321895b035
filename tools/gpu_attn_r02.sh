mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_ranker.py tests/test_gpu_attention_bwd.py tests/test_gpu_train.py -q -p no:cacheprovider -x > gpurun_out/attn_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/attn_tests.log
timeout -s KILL 120 python tools/probe_attn.py 2>&1 | tail -6
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attention_fwd -s 1 -c 1 -o gpurun_out/attn_r02 python tools/attn_once.py 2048 512 > /dev/null 2>&1; echo "ncu rc=$?"

mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_ranker.py -q -p no:cacheprovider -x -k "attention or small or full_depth" > gpurun_out/attn_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/attn_tests.log
timeout -s KILL 120 python tools/probe_attn.py 2>&1 | tail -6

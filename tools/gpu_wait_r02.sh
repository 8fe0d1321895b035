mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_ranker.py tests/test_gpu_attention_bwd.py tests/test_gpu_gemm.py tests/test_gpu_train.py -q -p no:cacheprovider -x > gpurun_out/wait_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/wait_tests.log
timeout -s KILL 120 python tools/probe_attn.py 2>&1 | tail -6
timeout -s KILL 120 python tools/probe_gemm.py 2>&1 | tail -8
timeout -s KILL 600 python bench.py --steps 3 --warmup 2 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks'], d['roofline']['frac'])"

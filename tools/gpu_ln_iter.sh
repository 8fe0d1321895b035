mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_ranker.py -q -p no:cacheprovider -x > gpurun_out/ln_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/ln_tests.log
for v in 1 0; do
  RSB200_LN_FUSED=$v timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fused=$v', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
done

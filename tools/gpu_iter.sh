# iteration run: build check, probes, targeted GPU tests, bench
mkdir -p gpurun_out
compute-sanitizer --tool synccheck tools/probes/mbar_tmem_synccheck > gpurun_out/probe_tmem_synccheck.log 2>&1; echo "probe2 rc=$?"; tail -4 gpurun_out/probe_tmem_synccheck.log
timeout 1800 python -m pytest -q -p no:cacheprovider -m gpu ${TESTS:-tests/test_gpu_tau.py tests/test_gpu_schedule.py} > gpurun_out/gputest_iter.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gputest_iter.log
if [ -n "${BENCH:-1}" ]; then timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_iter.err; fi

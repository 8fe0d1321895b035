mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_schedule.py tests/test_gpu_engine.py tests/test_gpu_cfg1.py -x > gpurun_out/gputest_engine.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_engine.log
timeout 300 python tools/engine_prof2.py 100000 20000 2>&1 | tail -1
timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -1
timeout 300 python tools/sort_lines.py 2>&1 | grep -E "rank_ms|rank_step"

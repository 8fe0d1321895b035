#!/bin/bash
# one-launch engine loop: engine tests, rank-step tests, A/B against the host loop
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_dropin.py -x -q > gpurun_out/gl_engine.log 2>&1; echo "engine rc=$?"
tail -3 gpurun_out/gl_engine.log
timeout 900 python -m pytest tests/test_gpu_schedule.py -x -q > gpurun_out/gl_sched.log 2>&1; echo "sched rc=$?"
tail -3 gpurun_out/gl_sched.log
timeout 1200 python tools/engine_ab.py 100000 > gpurun_out/gl_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/gl_ab.log | tail -5

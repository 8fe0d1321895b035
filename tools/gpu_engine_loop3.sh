#!/bin/bash
# engine loop: tests, A/B vs host loop, phase breakdown
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_dropin.py tests/test_gpu_schedule.py -x -q 2>&1 | tail -2
timeout 1200 python tools/engine_ab.py 100000 2>&1 | tail -4
RS_ENGINE_PROF=1 timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -16

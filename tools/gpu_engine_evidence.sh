#!/bin/bash
# engine loop evidence: A/B vs the host loop (identical rows / metrics), phase breakdown,
# one ncu --set full capture of the one-launch loop kernel (20k-request prefix)
mkdir -p gpurun_out
timeout 1200 python tools/engine_ab.py 100000 > gpurun_out/engine_ab.log 2>&1; echo "ab rc=$?"; tail -3 gpurun_out/engine_ab.log
RS_ENGINE_PROF=1 timeout 300 python tools/engine_prof2.py 100000 > gpurun_out/engine_phases.log 2>&1; tail -16 gpurun_out/engine_phases.log
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:engine_loop -c 1 -o gpurun_out/engloop_final python tools/engine_prof2.py 20000 > /dev/null 2>&1; echo "ncu rc=$?"

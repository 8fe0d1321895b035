#!/bin/bash
# engine loop phase breakdown at 8 / 16 / 4 CTAs
mkdir -p gpurun_out
for c in 8 16 4; do
  echo "CTAS=$c"; RS_ENGINE_CTAS=$c RS_ENGINE_PROF=1 timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -7
done

#!/bin/bash
# engine loop: speculative margin and cluster size sweep (us/step)
for mg in 256 128 64; do echo "margin=$mg"; RS_ENGINE_MARGIN=$mg timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -1; done
echo "ctas=16"; RS_ENGINE_CTAS=16 timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -1
echo "ctas=16 margin 128"; RS_ENGINE_MARGIN=128 RS_ENGINE_CTAS=16 timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -1
RS_ENGINE_MARGIN=128 RS_ENGINE_PROF=1 timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -16

#!/bin/bash
# rank step 1M: multi-launch (default) vs one-launch cluster of 16 / 8, and cooperative
echo default; timeout 300 python tools/sort_lines.py 2>&1 | grep -E "rank_ms"
echo "cl16 to 1M"; RS_SEL_FUSED_N=1048576 RS_SEL_CLUSTER_N=1048576 RS_SEL_CLUSTER=16 timeout 300 python tools/sort_lines.py 2>&1 | grep -E "rank_ms"
echo "cl8 to 1M"; RS_SEL_FUSED_N=1048576 RS_SEL_CLUSTER_N=1048576 RS_SEL_CLUSTER=8 timeout 300 python tools/sort_lines.py 2>&1 | grep -E "rank_ms"
echo "coop to 1M"; RS_SEL_FUSED_N=1048576 timeout 300 python tools/sort_lines.py 2>&1 | grep -E "rank_ms"
RS_SEL_FUSED_N=1048576 RS_SEL_CLUSTER_N=1048576 RS_SEL_CLUSTER=16 timeout 600 python -m pytest tests/test_gpu_schedule.py -x -q 2>&1 | tail -2

for v in 262144 1048576; do echo "FUSED_N=$v"; RS_SEL_FUSED_N=$v timeout 300 python tools/sort_lines.py 2>&1 | grep -E "rank_ms"; done

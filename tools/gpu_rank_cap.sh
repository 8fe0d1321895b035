mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:"sel_hist|sel_sort_emit" -c 3 -o gpurun_out/rank64m_full python tools/prof_sort.py rank 67108864 1 > /dev/null 2>&1; echo "ncu rc=$?"

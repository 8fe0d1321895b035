mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:tf_leaf -c 1 -o gpurun_out/leaf16m python tools/prof_sort.py tau 16777216 1 > /dev/null 2>&1; echo "leaf rc=$?"

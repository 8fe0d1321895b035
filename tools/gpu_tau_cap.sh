mkdir -p gpurun_out
for cap in 1024 2048 4096 8192; do for n in 1048576 67108864; do
  RS_TAU_CAP=$cap ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:tf_ \
      --log-file gpurun_out/cap_${cap}_$n.csv python tools/prof_sort.py tau $n 1 > gpurun_out/cap_${cap}_$n.out 2>&1
done; done
cat gpurun_out/cap_*_1048576.out | grep tau

mkdir -p gpurun_out
for spec in "tau 1048576" "tau 67108864" "rank 1048576" "rank 67108864"; do
  set -- $spec
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/prof_$1_$2.csv python tools/prof_sort.py $1 $2 3 > /dev/null 2>&1
  echo "$spec rc=$?"
done

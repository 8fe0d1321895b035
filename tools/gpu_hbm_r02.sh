# round-2 HBM-side evidence: per-kernel time + DRAM bytes for tau / rank step at 1M, 16M, 256M (64M rank),
# full captures of the tau leaf walk and ListMLE
mkdir -p gpurun_out
for spec in "tau 1048576" "tau 16777216" "tau 268435456" "rank 1048576" "rank 67108864"; do
  set -- $spec
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/prof_$1_$2.csv python tools/prof_sort.py $1 $2 2 > /dev/null 2>&1
  echo "$spec rc=$?"
done
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:tf_leaf -c 1 -o gpurun_out/leaf16m python tools/prof_sort.py tau 16777216 1 > /dev/null 2>&1; echo "leaf rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:listmle_lengths64 -c 1 -o gpurun_out/listmle_full python tools/listmle_once.py > /dev/null 2>&1; echo "listmle rc=$?"
timeout 300 python tools/sort_lines.py > gpurun_out/sort_lines.txt 2>&1; echo "lines rc=$?"
cat gpurun_out/sort_lines.txt

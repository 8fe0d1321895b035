mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_tau.py -x > gpurun_out/gputest_tau.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest_tau.log
for spec in "tau 1048576" "tau 67108864" "tau 268435456"; do
  set -- $spec
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/prof_$1_$2.csv python tools/prof_sort.py $1 $2 2 > /dev/null 2>&1
  echo "$spec rc=$?"
done
if [ -n "$LEAF" ]; then
  ncu --set full --clock-control none --import-source on -k regex:tf_leaf -c 1 -o gpurun_out/leaf64m python tools/prof_sort.py tau 67108864 1 > gpurun_out/leaf64m.log 2>&1; echo "ncu leaf rc=$?"
fi

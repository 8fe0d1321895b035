mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_schedule.py tests/test_gpu_engine.py tests/test_gpu_cfg1.py tests/test_gpu_tau.py -x > gpurun_out/gputest_rank.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_rank.log
for spec in "rank 1048576" "rank 67108864" "tau 1048576"; do
  set -- $spec
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/prof_$1_$2.csv python tools/prof_sort.py $1 $2 2 > /dev/null 2>&1
  echo "$spec rc=$?"
done

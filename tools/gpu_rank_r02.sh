# rank-step iteration: parity tests, bench lines, per-kernel times at 1M / 64M
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_schedule.py -x > gpurun_out/gputest_rank.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_rank.log
timeout 300 python tools/sort_lines.py 2>&1 | grep -E "rank"
for n in 1048576 67108864; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/prof_rank_$n.csv python tools/prof_sort.py rank $n 2 > /dev/null 2>&1
  echo "rank $n rc=$?"
done

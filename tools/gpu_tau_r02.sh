# tau iteration: parity tests, bench lines, per-kernel times at 16M / 256M
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_tau.py -x > gpurun_out/gputest_tau.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_tau.log
timeout 300 python tools/sort_lines.py 2>&1 | grep -E "tau"
for n in 16777216 268435456; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/prof_tau_$n.csv python tools/prof_sort.py tau $n 2 > /dev/null 2>&1
  echo "tau $n rc=$?"
done

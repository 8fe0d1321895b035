# round-2 end-of-session evidence: all GPU tests, the default bench, the reference arm,
# a launch list of one step
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest_final.log
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo "ref rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1; echo "ncu rc=$?"
python -c "import smoke_check" 2>/dev/null; python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"

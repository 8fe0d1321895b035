# round-2 closing evidence (re-entry session): all GPU tests, smoke, default bench,
# reference arm, launch list of one headline step
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final4.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputest_final4.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest_final4.log
timeout 1200 python bench.py > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final4.json 2> gpurun_out/bench_ref_final4.err; echo "ref rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final4.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1; echo "ncu rc=$?"

# round-2 re-entry check: all GPU tests + smoke + default bench on HEAD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_re.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputest_re.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/gputest_re.log
timeout 1200 python bench.py > gpurun_out/bench_re.json 2> gpurun_out/bench_re.err; echo "bench rc=$?"

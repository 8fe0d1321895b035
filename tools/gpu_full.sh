# full round check: all GPU tests, then the default bench, then the reference arm
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_full.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/gputest_full.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_full.csv &
CLK=$!
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
kill $CLK
tail -3 gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"

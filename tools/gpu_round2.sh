# round-2 evidence pass: all GPU tests, default bench, reference arm, launch list of one step
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest_full.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest_full.log
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-extras > gpurun_out/bench_ncu.json 2>&1; echo "ncu rc=$?"
cat gpurun_out/bench_full.json gpurun_out/bench_ref.json

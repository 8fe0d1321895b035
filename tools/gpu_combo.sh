mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_train.py tests/test_gpu_ranker.py -q -p no:cacheprovider --timeout 120 --timeout-method thread -rf > gpurun_out/train.log 2>&1
grep -v "^  File\|^    " gpurun_out/train.log | grep -v "^$" | tail -30
timeout -s KILL 120 python tools/attn_trace.py > gpurun_out/attn_trace.log 2>&1; cat gpurun_out/attn_trace.log
timeout -s KILL 120 python tools/probe_attn.py > gpurun_out/probe_attn.log 2>&1; cat gpurun_out/probe_attn.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json

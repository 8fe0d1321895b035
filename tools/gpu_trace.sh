mkdir -p gpurun_out
timeout -s KILL 120 python tools/attn_trace.py > gpurun_out/attn_trace.log 2>&1; cat gpurun_out/attn_trace.log

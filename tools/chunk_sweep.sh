# Forward throughput vs activation chunk size (tokens per slice) — L2 residency sweep.
for t in 1048576 262144 131072 65536 32768 16384; do
  RSB200_CHUNK_TOKENS=$t timeout 300 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/chunk_$t.json 2>&1
  python - "$t" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/chunk_{t}.json").read().strip().splitlines()[-1])
    print(t, round(d["value"]), d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(t, "failed", e)
PY
done

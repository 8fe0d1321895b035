mkdir -p gpurun_out
for shp in "fwd 2 100 4" "bwd 1 128 1" "bwd 3 64 12" "bwd 1 100 1" "bwd 2 100 1" "bwd 2 128 4" "bwd 2 64 4" "bwd 2 96 4" "bwd 2 100 4" "bwd 1 127 1"; do
  echo "== $shp"; timeout -s KILL 40 python tools/probe_bwd.py $shp 2>&1 | tail -3
done > gpurun_out/probe.log 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_train.py -q -p no:cacheprovider -k "64-16-4-2 or 128-8-3-3 or adam or deterministic" --timeout 120 --timeout-method thread -rf -x > gpurun_out/train.log 2>&1
cat gpurun_out/probe.log; grep -v "^  File\|^    " gpurun_out/train.log | tail -40

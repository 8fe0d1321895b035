mkdir -p gpurun_out
for shp in "bwd 1 100 1" "bwd 2 100 4" "bwd 1 127 1" "bwd 3 33 2"; do
  echo "== $shp"; timeout -s KILL 40 python tools/probe_bwd.py $shp 2>&1 | tail -3
done > gpurun_out/probe.log 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_train.py tests/test_gpu_attention_bwd.py -q -p no:cacheprovider --timeout 120 --timeout-method thread -rf > gpurun_out/train.log 2>&1
cat gpurun_out/probe.log; grep -v "^  File\|^    " gpurun_out/train.log | grep -v "^$" | tail -40

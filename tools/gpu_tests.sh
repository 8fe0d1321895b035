# Run every GPU test file separately, each bounded, so one hang cannot eat the call.
mkdir -p gpurun_out
for f in tests/test_gpu_*.py; do
  b=$(basename $f .py)
  timeout -s KILL ${FILE_TIMEOUT:-600} python -m pytest $f -q -p no:cacheprovider --timeout ${TEST_TIMEOUT:-180} --timeout-method thread -rf > gpurun_out/$b.log 2>&1
  echo "$b rc=$? $(tail -1 gpurun_out/$b.log)"
done

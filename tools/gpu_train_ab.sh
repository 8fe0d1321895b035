mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention_bwd.py tests/test_gpu_train.py -q -x -p no:cacheprovider > gpurun_out/train_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/train_tests.log
for k in 1 2; do
echo "old S512"; RSB200_LIB=$PWD/tools/_ab/librsb200_old.so timeout 600 python tools/train_time.py 64 512 2>&1 | tail -1
echo "new S512"; timeout 600 python tools/train_time.py 64 512 2>&1 | tail -1
done

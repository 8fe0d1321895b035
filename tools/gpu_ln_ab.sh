mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py -q -x -p no:cacheprovider > gpurun_out/ln_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ln_tests.log
for k in 1 2; do
echo "old S128"; RSB200_LIB=$PWD/tools/_ab/librsb200_old.so timeout 600 python tools/train_time.py 1024 128 2>&1 | tail -1
echo "new S128"; timeout 600 python tools/train_time.py 1024 128 2>&1 | tail -1
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:ln_bwd --log-file gpurun_out/lnb_new.csv python tools/train_once.py 16 16 > /dev/null 2>&1
RSB200_LIB=$PWD/tools/_ab/librsb200_old.so timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:ln_bwd --log-file gpurun_out/lnb_old.csv python tools/train_once.py 16 16 > /dev/null 2>&1
echo done

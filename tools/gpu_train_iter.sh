mkdir -p gpurun_out
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_train.py tests/test_gpu_train_ranking.py tests/test_gpu_classifier.py tests/test_gpu_gemm.py -x > gpurun_out/gputest_train.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_train.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_train.csv python tools/train_once.py 16 16 > /dev/null 2>&1; echo "train rc=$?"
timeout 900 python tools/train_time.py 1024 128 2>&1 | tail -1

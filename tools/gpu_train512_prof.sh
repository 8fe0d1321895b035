mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_train512.csv python tools/train_once.py 4 4 512 > gpurun_out/train512.log 2>&1; echo "train rc=$?"

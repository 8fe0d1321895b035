# one training micro-batch (16 lists x 64 x 128 tokens): per-kernel time + DRAM bytes
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_train.csv python tools/train_once.py 16 16 > /dev/null 2>&1; echo "train rc=$?"

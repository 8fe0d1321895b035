# one ncu --set full capture of a kernel: KERNEL=regex WHAT="tau 1048576" OUT=name
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:${KERNEL} -s ${SKIP:-0} -c ${COUNT:-1} \
    -o gpurun_out/${OUT} python tools/prof_sort.py ${WHAT} 2 > gpurun_out/${OUT}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${OUT}.log

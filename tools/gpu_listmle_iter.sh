# ListMLE iteration: parity tests, timing, full capture
mkdir -p gpurun_out
timeout 600 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_listmle.py tests/test_gpu_properties.py -x > gpurun_out/gputest_listmle.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_listmle.log
python tools/listmle_once.py
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:listmle_lengths64 -c 1 -o gpurun_out/listmle_full2 python tools/listmle_once.py > /dev/null 2>&1; echo "ncu rc=$?"

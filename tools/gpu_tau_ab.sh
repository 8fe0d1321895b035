mkdir -p gpurun_out
timeout 600 python tools/tau_ab.py > gpurun_out/tau_ab.log 2>&1; echo "ab rc=$?"; grep -v "^ok" gpurun_out/tau_ab.log | tail -12
timeout 900 python -m pytest tests/test_gpu_tau.py tests/test_gpu_properties.py -q -x -p no:cacheprovider > gpurun_out/tau_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tau_tests.log
echo "--- old lib"; RSB200_LIB=$PWD/tools/_ab/librsb200_old.so timeout 600 python tools/tau_ab.py --time-only 2>&1 | tail -7
echo "--- new lib"; timeout 600 python tools/tau_ab.py --time-only 2>&1 | tail -7
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tau1m_new.csv python tools/tau_once.py > /dev/null 2>&1; echo "ncu rc=$?"
RSB200_LIB=$PWD/tools/_ab/librsb200_old.so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tau1m_old.csv python tools/tau_once.py > /dev/null 2>&1; echo "ncu rc=$?"

mkdir -p gpurun_out
for rm in 48 0; do echo "--- check RS_TAU_RANK_MAX=$rm"; RS_TAU_RANK_MAX=$rm timeout 600 python tools/tau_ab.py --check-only 2>&1 | grep -v "^ok" | tail -5; done
timeout 900 python -m pytest tests/test_gpu_tau.py tests/test_gpu_properties.py -q -x -p no:cacheprovider > gpurun_out/tau_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tau_tests.log
echo "--- old lib"; RSB200_LIB=$PWD/tools/_ab/librsb200_old.so timeout 600 python tools/tau_ab.py --time-only 2>&1 | tail -7
for rm in 0 24 48 96; do echo "--- new lib rank_max=$rm"; RS_TAU_RANK_MAX=$rm timeout 600 python tools/tau_ab.py --time-only 2>&1 | tail -7; done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tau1m_new2.csv python tools/tau_once.py > /dev/null 2>&1; echo "ncu rc=$?"

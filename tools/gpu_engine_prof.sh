mkdir -p gpurun_out
timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -1
timeout 300 python tools/engine_prof2.py 100000 20000 2>&1 | tail -1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 40000 -c 2000 --csv --log-file gpurun_out/engine_launches.csv python tools/engine_prof2.py 100000 20000 > /dev/null 2>&1; echo "ncu rc=$?"

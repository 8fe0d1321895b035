mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:tf_leaf -c 1 -o gpurun_out/leaf1m python tools/tau_once.py > gpurun_out/leaf_prof.log 2>&1; echo "ncu rc=$?"

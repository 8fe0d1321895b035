# Full ncu captures of the HBM-side kernels of the sort / tau / loss rows:
# ListMLE (1M lists x 64), a tau merge pass and the histogram count pass at 16M, the
# rank-step select histogram and state update at 16M.
mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:listmle_lengths64 -c 1 -o gpurun_out/hbm_listmle python tools/listmle_once.py > /dev/null 2>&1; echo "listmle rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none -k regex:"ms_merge_pass|chunk_cross" -s 4 -c 2 -o gpurun_out/hbm_tau python tools/tau_big.py 16777216 > /dev/null 2>&1; echo "tau rc=$?"
timeout -s KILL 300 ncu --set full --clock-control none -k regex:"sel_hist|starvation_update|build_rank_keys" -c 3 -o gpurun_out/hbm_rank python tools/rank_once.py 16777216 > /dev/null 2>&1; echo "rank rc=$?"
ls -la gpurun_out/hbm_*

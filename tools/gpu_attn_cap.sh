mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attention_fwd -s 1 -c 1 -o gpurun_out/attn_r02 python tools/attn_once.py 2048 512 > /dev/null 2>&1; echo "ncu rc=$?"

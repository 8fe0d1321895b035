mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attention -s 1 -c 1 -o gpurun_out/attn2 python tools/attn_once.py 2048 512 > gpurun_out/ncu_attn2.log 2>&1
ls gpurun_out

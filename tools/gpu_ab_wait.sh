# A/B on one box: forward step with the sleeping mbarrier wait (current) vs the spinning one
mkdir -p gpurun_out
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"; }
run new; run new
cp paper_2408_15792_b200/csrc/sm100.cuh /tmp/sm100_new.cuh
cp tools/probes/sm100_old.cuh.txt paper_2408_15792_b200/csrc/sm100.cuh
make -s -j16 -C paper_2408_15792_b200/csrc > /dev/null 2>&1; echo "make rc=$?"
run old; run old
cp /tmp/sm100_new.cuh paper_2408_15792_b200/csrc/sm100.cuh
make -s -j16 -C paper_2408_15792_b200/csrc > /dev/null 2>&1
run new; run new

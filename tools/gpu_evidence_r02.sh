# Round-2 ncu evidence for profiles/ (one GPU, never multi-rank): per-call DRAM bytes of the
# cfg4 tau / rank step, --set full captures of the dominant kernel of every bench line.
mkdir -p gpurun_out/ev
M=$((1<<20))
T="timeout -s KILL 300"
MET="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
$T ncu $MET --log-file gpurun_out/ev/tau1m.csv python tools/tau_once.py > /dev/null 2>&1; echo "tau1m rc=$?"
$T ncu $MET --log-file gpurun_out/ev/rank1m.csv python tools/rank_once.py > /dev/null 2>&1; echo "rank1m rc=$?"
$T ncu $MET --log-file gpurun_out/ev/rank64m.csv python tools/rank_once.py 67108864 > /dev/null 2>&1; echo "rank64m rc=$?"
$T ncu $MET --log-file gpurun_out/ev/tau256m.csv python tools/tau_big.py 268435456 > /dev/null 2>&1; echo "tau256m rc=$?"
FULL="--set full --clock-control none --import-source on"
for spec in "qkv 2304 768 7" "out 768 768 2" "fc1 3072 768 1" "fc2 768 3072 2"; do
  set -- $spec
  $T ncu $FULL -k regex:gemm_bf16_2sm -s 1 -c 1 -o gpurun_out/ev/gemm_$1 python tools/gemm_once.py $M $2 $3 $4 > /dev/null 2>&1; echo "gemm $1 rc=$?"
done
$T ncu $FULL -k regex:attention_fwd -s 1 -c 1 -o gpurun_out/ev/attn python tools/attn_once.py 2048 512 > /dev/null 2>&1; echo "attn rc=$?"
$T ncu $FULL -k regex:layernorm_kernel -c 1 -o gpurun_out/ev/layernorm python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1; echo "ln rc=$?"
$T ncu $FULL -k regex:listmle_lengths64 -c 1 -o gpurun_out/ev/listmle python tools/listmle_once.py > /dev/null 2>&1; echo "listmle rc=$?"
$T ncu $FULL -k regex:tf_leaf -c 1 -o gpurun_out/ev/tau_leaf_1m python tools/tau_once.py > /dev/null 2>&1; echo "leaf rc=$?"
$T ncu $FULL -k regex:"sel_hist|starvation_update_v" -c 3 -o gpurun_out/ev/rank64m python tools/rank_once.py 67108864 > /dev/null 2>&1; echo "rank rc=$?"
$T ncu $FULL -k regex:"gemm_bf16_2sm_kernel<6" -c 1 -o gpurun_out/ev/wgrad python tools/train_once.py 16 16 > /dev/null 2>&1; echo "wgrad rc=$?"
ls gpurun_out/ev

# Attention exponential split sweep: one library per MUFU mask (variants/, built locally
# with -DAT_MUFU_MASK=...), timed by tools/probe_attn.py on the same box.
for m in 0x57 0x55 0x5F 0x77 0xFF; do
  echo "mask $m"; RSB200_LIB=variants/librsb200_$m.so python tools/probe_attn.py 2>&1 | grep "B=2048 reps=10"
done

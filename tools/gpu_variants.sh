for m in 0x55 0x57 0x15 0x77 0x11; do
  echo "mask $m"; RSB200_LIB=variants/librsb200_$m.so python tools/probe_attn.py 2>&1 | grep "B=2048 reps=10"
done

for v in 16384 8192 4096 2048; do
  echo "SEL_MIN_N=$v"; RS_SEL_MIN_N=$v timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -1
done

for v in 262144 65536 16384 4096; do
  echo "SEL_MIN_N=$v"; RS_SEL_MIN_N=$v timeout 300 python tools/engine_prof2.py 100000 20000 2>&1 | tail -1
done

for n in ${SIDES:-40 64 96 128 148}; do
  echo "== side_ctas $n"
  PDIPC_SIDE_CTAS=$n PDIPC_TIMELINE=1 timeout 300 python tools/timeline_c2.py 25 1 2>&1 | sed -n '8p;$p'
done

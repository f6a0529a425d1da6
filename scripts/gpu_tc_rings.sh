# Sweep tc_dots ring depths (A, TMEM A slots, X) at the C4 shape (timing experiments).
for r in ${RINGS:-10,2,3 8,2,5 10,3,3 10,4,3 6,2,6}; do
  for pr in ${PROBES:-0 16}; do
    echo -n "rings=$r "; GPSPCA_TC_RINGS=$r GPSPCA_TC_PROBE=$pr TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
  done
done

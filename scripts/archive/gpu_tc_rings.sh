# Sweep tc_dots ring depths ("A,X" stages) and TMEM segment lengths at C3- and
# C4-like shapes (timing experiments; GPSPCA_TC_RINGS / GPSPCA_TC_SEG).
for r in 5,3 6,3 6,2 4,3 3,3; do
  echo -n "C3 rings=$r "; TC_P=4096 TC_M=10 TC_N=1048576 GPSPCA_TC_RINGS=$r TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
done
for r in 5,3 4,3 5,2 4,4 3,3; do
  echo -n "C4 rings=$r "; TC_P=8192 TC_M=64 TC_N=524288 GPSPCA_TC_RINGS=$r TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
done
for sg in 1 2 4 8; do
  echo -n "C4 seg=$sg "; TC_P=8192 TC_M=64 TC_N=524288 GPSPCA_TC_SEG=$sg TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
  echo -n "C3 seg=$sg "; TC_P=4096 TC_M=10 TC_N=1048576 GPSPCA_TC_SEG=$sg TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
done

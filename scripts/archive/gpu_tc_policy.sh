# T1 A-stream experiments: L2 cache hint on the A boxes (probe 128 drops
# evict_first) and the tensor map's L2 promotion (GPSPCA_TC_APROMO).
for pr in 0 128; do for promo in 256 128 0; do
  echo -n "C3 probe=$pr promo=$promo "; TC_P=4096 TC_M=10 TC_N=1048576 GPSPCA_TC_PROBE=$pr GPSPCA_TC_APROMO=$promo TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
  echo -n "C4 probe=$pr promo=$promo "; TC_P=8192 TC_M=64 TC_N=524288 GPSPCA_TC_PROBE=$pr GPSPCA_TC_APROMO=$promo TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
done; done

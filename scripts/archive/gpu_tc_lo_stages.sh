for lib in libgpspca_b200.so libgpspca_b200_lo3.so libgpspca_b200_lo4.so; do for rep in 1 2; do
  echo -n "$lib C3 "; GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib TC_P=4096 TC_M=10 TC_N=1048576 TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
  echo -n "$lib C4 "; GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib TC_P=8192 TC_M=64 TC_N=524288 TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
done; done

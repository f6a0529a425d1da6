# SU sweep: evict_first vs evict_normal on the A bulk stream (diagnostics
# build paper_1312_6182_b200/libgpspca_b200_evn.so, GPS_STREAM_EVICT_NORMAL).
for lib in libgpspca_b200.so libgpspca_b200_evn.so; do for rep in 1 2; do
  echo "lib=$lib"; GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib timeout 300 python bench.py --steps 100 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['read_stream_gbs'])"
done; done
for lib in libgpspca_b200.so libgpspca_b200_evn.so; do
  echo -n "C3 lib=$lib "; GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib TC_P=4096 TC_M=10 TC_N=1048576 TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
done

# A/B of the fused single-unit sweep: paper_1312_6182_b200/libgpspca_b200_base.so
# vs variant builds (VARIANTS="libgpspca_b200_x.so ..."), alternating, C2
# headline only, plus the gamma = 0 dense probe.
mkdir -p gpurun_out
V=${VARIANTS:-libgpspca_b200.so}
for rep in 1 2 3; do
  for lib in libgpspca_b200_base.so $V; do
    GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib timeout 600 python bench.py --steps 300 --e2e-steps 0 --no-cpu-baseline --no-block 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), 'it/s', round(d['roofline']['achieved']), 'GB/s sweep', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
for lib in libgpspca_b200_base.so $V; do
  GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib timeout 300 python scripts/su_dense_probe.py 0 20 2>&1 | tail -1 | sed "s/^/$lib gamma0: /"
done

# A/B of the fused single-unit sweep: HEAD library vs a baseline build
# (paper_1312_6182_b200/libgpspca_b200_base.so), alternating, C2 headline
# only, plus the gamma = 0 dense probe; then the single-unit parity suites.
mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in libgpspca_b200_base.so libgpspca_b200.so; do
    GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib timeout 600 python bench.py --steps 300 --e2e-steps 0 --no-cpu-baseline --no-block 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), 'it/s', round(d['roofline']['achieved']), 'GB/s sweep', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
for lib in libgpspca_b200_base.so libgpspca_b200.so; do
  GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib timeout 300 python scripts/su_dense_probe.py 0 20 2>&1 | tail -1 | sed "s/^/$lib gamma0: /"
done
timeout 1200 python -m pytest tests/test_gpu_single_unit.py tests/test_gpu_acceptance.py tests/test_gpu_scale.py tests/test_gpu_band.py \
  tests/test_gpu_peer_exchange.py "tests/test_gpu_fullsize.py::test_c2_full_solve" "tests/test_gpu_fullsize.py::test_c2_gamma0_trajectory" \
  -x -q -p no:cacheprovider 2>&1 | tail -3

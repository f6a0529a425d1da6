mkdir -p gpurun_out
for lib in libgpspca_b200.so libgpspca_b200_k2.so; do
  for rep in 1 2; do
    GPSPCA_LIB=$PWD/paper_1312_6182_b200/$lib timeout 600 python bench.py --steps 200 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['roofline']['achieved']), round(d['roofline']['read_stream_gbs']), d['clocks'])"
  done
done

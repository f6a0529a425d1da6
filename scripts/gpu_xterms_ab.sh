# One- vs two-term X in T1 (GPSPCA_TC_XTERMS): block parity suites, sustained
# C4 sweeps with clocks, the bench's block lines.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_block.py tests/test_gpu_block_large.py tests/test_gpu_hard.py tests/test_gpu_threshold_band.py tests/test_gpu_band.py -x -q -p no:cacheprovider 2>&1 | tail -2
for xt in 1 2 1 2; do GPSPCA_TC_XTERMS=$xt ITERS=60 timeout 300 python scripts/c4_power_probe.py 2>&1 | tail -1 | sed "s/^/xterms=$xt /"; done
for xt in 1 2; do
  GPSPCA_TC_XTERMS=$xt timeout 900 python bench.py --steps 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('xterms=$xt', {k: (round(v['iters_per_s'],1), round(v['ms_per_iter'],3), v['clocks']['sm_mhz'], v['clocks']['reasons']) for k,v in d['block_configs'].items()})"
done

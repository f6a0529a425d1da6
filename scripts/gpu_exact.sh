# Exact fp32 block path (T1 filter + T1x recomputation): block parity suites,
# smoke, per-iteration times at C3 / C4 and the ncu launch split.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_block_large.py tests/test_gpu_scale.py tests/test_gpu_distributed_world2.py -q -x > gpurun_out/tb.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/tb.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
for cfg in c3 c4; do for data in gauss planted; do
  TC_CFG=$cfg TC_DATA=$data timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -2
done; done
TC_CFG=c3 TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c3_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
TC_CFG=c4 TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c4_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log

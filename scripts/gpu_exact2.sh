# Exact tensor-core block path (fp32 + fp64): full GPU suite, smoke, C3 / C4
# iteration times and ncu launch splits.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
for cfg in c3 c4; do for data in gauss planted; do
  TC_CFG=$cfg TC_DATA=$data timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1
done; done
TC_CFG=c3 TC_DATA=planted TC_DTYPE=f64 timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1
GPSPCA_NO_TC=1 TC_CFG=c3 TC_DATA=planted TC_DTYPE=f64 timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1
TC_CFG=c3 TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c3_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
TC_CFG=c4 TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c4_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"

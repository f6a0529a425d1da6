# Refinement kernel variants: block parity suites + C3 / C4 launch splits,
# and a denser-activity probe (gamma = 0.03 max ||a_i||).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_block_large.py tests/test_gpu_scale.py -q -x > gpurun_out/tb.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tb.log
for cfg in c3 c4; do TC_CFG=$cfg TC_DATA=planted timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1; done
TC_CFG=c3 TC_DATA=gauss TC_GFRAC=0.05 timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1
TC_CFG=c3 TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c3_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
TC_CFG=c4 TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c4_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
TC_CFG=c3 TC_DATA=gauss TC_GFRAC=0.05 TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c3d_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c3d.log 2>&1; echo "ncu c3d rc=$?"
python scripts/launch_split.py gpurun_out/exact_c3_launches.csv gpurun_out/exact_c4_launches.csv gpurun_out/exact_c3d_launches.csv

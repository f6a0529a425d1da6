mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_block_large.py tests/test_gpu_scale.py tests/test_gpu_distributed_world2.py -q -x > gpurun_out/tb.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tb.log
for cfg in c3 c4; do TC_CFG=$cfg TC_DATA=planted timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1; done
TC_CFG=c3 TC_DATA=gauss TC_GFRAC=0.05 timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1
TC_CFG=c3 TC_DATA=gauss TC_GFRAC=0.05 TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c3d_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c3d.log 2>&1; echo "ncu c3d rc=$?"
python scripts/launch_split.py gpurun_out/exact_c3d_launches.csv | grep -v "bk_\|gram\|chol\|apply"
for pr in 0 8 4 32 44; do
  echo -n "C3 "; TC_P=4096 TC_M=10 TC_N=1048576 GPSPCA_TC_PROBE=$pr TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
  echo -n "C4 "; TC_P=8192 TC_M=64 TC_N=524288 GPSPCA_TC_PROBE=$pr TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -1
done

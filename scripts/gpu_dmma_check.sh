# DMMA refine / update kernels: block parity suites, C4 dense timing and launch split
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_hard.py tests/test_gpu_block_large.py tests/test_gpu_threshold_band.py tests/test_gpu_band.py -m gpu -q -x > gpurun_out/dmma_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/dmma_tests.log
for cfg in "c4 gauss 0.03" "c4 planted 0.1" "c3 gauss 0.05" "c3 planted 0.1"; do set -- $cfg
  TC_CFG=$1 TC_DATA=$2 TC_GFRAC=$3 TC_ITERS=4 timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1 >> gpurun_out/dmma_times.log; done
TC_CFG=c4 TC_DATA=gauss TC_GFRAC=0.03 TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c4d_launches_dmma.csv python scripts/tc_breakdown.py > gpurun_out/c4d_ncu_dmma.log 2>&1
python scripts/launch_split.py gpurun_out/c4d_launches_dmma.csv >> gpurun_out/dmma_times.log

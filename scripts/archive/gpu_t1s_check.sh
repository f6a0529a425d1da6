mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_hard.py tests/test_gpu_threshold_band.py -x -q -p no:cacheprovider 2>&1 | tail -2
bash scripts/gpu_small_n_split.sh 2>&1 | grep -E "median|refine|update|dots"
T1X_CFG=C4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/t1x_candidates.py > /dev/null 2>&1; python scripts/launch_split.py gpurun_out/c4_launches.csv | grep -E "refine"

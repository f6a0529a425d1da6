# Cross-process IPC exchange test, T1x candidate distribution and per-iteration
# times at the bench's block configurations.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_px_ipc.py tests/test_gpu_peer_exchange.py -x -q -p no:cacheprovider > gpurun_out/px_ipc.log 2>&1; echo "px rc=$?"
for c in C3 C4 C4_dense; do
  T1X_CFG=$c GPSPCA_TC_PROBE=512 timeout 300 python scripts/t1x_candidates.py >> gpurun_out/t1x.log 2>&1
  T1X_CFG=$c timeout 300 python scripts/t1x_candidates.py >> gpurun_out/t1x.log 2>&1
done
T1X_CFG=C4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/t1x_candidates.py > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/launch_split.py gpurun_out/c4_launches.csv > gpurun_out/c4_split.txt 2>&1
tail -5 gpurun_out/px_ipc.log; cat gpurun_out/t1x.log; cat gpurun_out/c4_split.txt

# Block-path parity suites + the C3 / C4 / dense-C4 iteration times and the
# C4 per-kernel split (after a change to the tensor-core block sweep).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_block.py tests/test_gpu_block_large.py tests/test_gpu_hard.py \
  tests/test_gpu_threshold_band.py tests/test_gpu_band.py tests/test_gpu_distributed_world2.py -x -q -p no:cacheprovider \
  > gpurun_out/block_tests.log 2>&1; echo "block tests rc=$?"; tail -3 gpurun_out/block_tests.log
rm -f gpurun_out/t1x.log
for c in C3 C4 C4_dense; do T1X_CFG=$c timeout 300 python scripts/t1x_candidates.py >> gpurun_out/t1x.log 2>&1; done
cat gpurun_out/t1x.log
T1X_CFG=C4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/t1x_candidates.py > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/launch_split.py gpurun_out/c4_launches.csv
( cd scripts/ubench && nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I ../../paper_1312_6182_b200/csrc polar_ns.cu -o polar_ns && ./polar_ns ) > gpurun_out/polar_ns.log 2>&1; cat gpurun_out/polar_ns.log

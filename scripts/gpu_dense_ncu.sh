# Dense-activity captures (round 2): K1 at gamma = 0 (every column active)
# and the fp64 recompute / update kernels of the tensor-core block path on
# C4 Gaussian data at gamma = (0.03 max ||a_i||)^2.
mkdir -p gpurun_out
python scripts/su_dense_probe.py 0 5 > gpurun_out/su_dense_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:su_sweep -s 2 -c 1 -o gpurun_out/su_dense \
      python scripts/su_dense_probe.py 0 5 > gpurun_out/su_dense_ncu.log 2>&1
echo "su rc=$?"
TC_CFG=c4 TC_DATA=gauss TC_GFRAC=0.03 TC_ITERS=3 python scripts/tc_breakdown.py > gpurun_out/c4d_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"tc_refine|tc_update" -s 2 -c 2 -o gpurun_out/c4_dense \
      env TC_CFG=c4 TC_DATA=gauss TC_GFRAC=0.03 TC_ITERS=3 python scripts/tc_breakdown.py > gpurun_out/c4d_ncu.log 2>&1
echo "c4 rc=$?"
TC_CFG=c4 TC_DATA=gauss TC_GFRAC=0.03 TC_ITERS=3 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c4d_launches.csv python scripts/tc_breakdown.py > gpurun_out/c4d_ncu2.log 2>&1
echo "split rc=$?"

# Round-2 evidence: bench lines (ours + reference arm), the C2 launch list and
# full capture of the headline sweep, the dense captures (K1 at gamma = 0,
# DMMA T1x / T2 on dense C4), and C3 / C4 launch splits.
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_r2.json 2> gpurun_out/bench_ref_r2.err; echo "ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-block"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:su_sweep -s 3 -c 1 -o gpurun_out/prof_sweep_r2 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu sweep rc=$?"
python scripts/su_dense_probe.py 0 5 > gpurun_out/su_dense_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:su_sweep -s 2 -c 1 -o gpurun_out/su_dense_r2 \
      python scripts/su_dense_probe.py 0 5 > gpurun_out/su_dense_ncu.log 2>&1; echo "ncu dense su rc=$?"
TC_CFG=c4 TC_DATA=gauss TC_GFRAC=0.03 TC_ITERS=3 timeout 600 python scripts/tc_breakdown.py > gpurun_out/c4d_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_refine|tc_update" -s 2 -c 2 -o gpurun_out/c4_dense_r2 \
      env TC_CFG=c4 TC_DATA=gauss TC_GFRAC=0.03 TC_ITERS=3 python scripts/tc_breakdown.py > gpurun_out/c4d_ncu.log 2>&1; echo "ncu dense c4 rc=$?"
for cfg in c3 c4; do
  TC_CFG=$cfg TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${cfg}_launches_r2.csv python scripts/tc_breakdown.py > gpurun_out/${cfg}_ncu_r2.log 2>&1; echo "ncu $cfg rc=$?"
done

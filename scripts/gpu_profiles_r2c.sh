# Block-path evidence at the final code: C3 / C4 per-kernel splits and one
# full capture of T1 at C4 (DRAM traffic, pipe utilisation, stalls).
mkdir -p gpurun_out
for cfg in C3 C4; do
  T1X_CFG=$cfg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${cfg}_launches_r2c.csv python scripts/t1x_candidates.py > /dev/null 2>&1; echo "ncu $cfg rc=$?"
done
T1X_CFG=C4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_dots -s 2 -c 1 -o gpurun_out/prof_t1_c4_r2c python scripts/t1x_candidates.py > gpurun_out/ncu_t1.log 2>&1; echo "ncu t1 rc=$?"
tail -3 gpurun_out/ncu_t1.log

# Round-2 closing evidence at HEAD: bench line (ours + reference arm), the C2
# launch list and one full capture of the headline sweep, the C4 per-kernel
# split.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_r2b.json 2> gpurun_out/bench_ref_r2b.err; echo "ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-block"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2b.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:su_sweep -s 3 -c 1 -o gpurun_out/prof_sweep_r2b $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu sweep rc=$?"
for cfg in C3 C4; do
  T1X_CFG=$cfg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${cfg}_launches_r2b.csv python scripts/t1x_candidates.py > /dev/null 2>&1; echo "ncu $cfg rc=$?"
done

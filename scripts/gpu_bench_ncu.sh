mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 python bench.py --steps 100 --warmup 5 --e2e-steps 2 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_full.err; cat gpurun_out/bench_full.json
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:su_sweep -s 3 -c 1 -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu_full.log

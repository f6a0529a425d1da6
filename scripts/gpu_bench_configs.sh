mkdir -p gpurun_out
timeout 900 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"
cat gpurun_out/bench_e2e.json; tail -3 gpurun_out/bench_e2e.err
timeout 1500 python scripts/bench_configs.py --tag r1 > gpurun_out/configs.log 2>&1; echo "configs rc=$?"
tail -40 gpurun_out/configs.log
cp profiles/configs_r1.jsonl gpurun_out/ 2>/dev/null

# quick iteration: GPU tests + bench (no e2e/cpu) + ncu full of the sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 python bench.py --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_iter.err; cat gpurun_out/bench_iter.json
if [ "${NCU:-1}" = "1" ]; then
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:su_sweep -s 3 -c 1 -o gpurun_out/prof_iter -f $CMD > gpurun_out/ncu_iter.log 2>&1; echo "ncu rc=$?"
fi

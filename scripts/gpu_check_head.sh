mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_head.json 2> gpurun_out/bench_head.err; echo "bench rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"
tail -40 gpurun_out/gputest.log

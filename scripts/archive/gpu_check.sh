mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 1 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json

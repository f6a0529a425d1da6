# Full GPU suite, smoke, C2 bench + reference arm, C3 / C4 iteration times.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-200
for cfg in c3 c4; do TC_CFG=$cfg TC_DATA=planted timeout 300 python scripts/tc_breakdown.py 2>&1 | tail -1; done

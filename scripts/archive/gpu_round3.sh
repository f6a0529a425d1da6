# Full GPU suite, smoke, C2 bench + reference arm, per-config sweep (C3 / C4 / C5),
# C3 / C4 launch splits of the block path.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python scripts/bench_configs.py --tag r1 > gpurun_out/cfg.log 2>&1; echo "configs rc=$?"; tail -40 gpurun_out/cfg.log
TC_CFG=c3 TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c3_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
TC_CFG=c4 TC_DATA=planted TC_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_c4_launches.csv python scripts/tc_breakdown.py > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
python scripts/launch_split.py gpurun_out/exact_c3_launches.csv gpurun_out/exact_c4_launches.csv

timeout 120 python scripts/tc_probe.py 2>&1 | tail -8
timeout 600 python scripts/bench_configs.py --only c4 --tag tc 2>&1 | tail -4

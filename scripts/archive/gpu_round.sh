# Full GPU suite, per-config sweep, C4 launch list (tensor-core block path).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/t.log
timeout 600 python scripts/bench_configs.py --tag r1 > gpurun_out/cfg.log 2>&1; echo "configs rc=$?"; cat gpurun_out/cfg.log | tail -20
python scripts/tc_c4_probe.py > gpurun_out/tc_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv python scripts/tc_c4_probe.py > gpurun_out/tc_ncu1.log 2>&1; echo "ncu1 rc=$?"
cat gpurun_out/tc_plain.log

# Full GPU suite, per-config sweep, C4 launch list + one full ncu capture of tc_dots.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/t.log
timeout 600 python scripts/bench_configs.py --tag r1 > gpurun_out/cfg.log 2>&1; echo "configs rc=$?"; tail -22 gpurun_out/cfg.log
timeout 300 python scripts/tc_c4_probe.py > gpurun_out/tc_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv python scripts/tc_c4_probe.py > gpurun_out/tc_ncu1.log 2>&1; echo "ncu1 rc=$?"
cat gpurun_out/tc_plain.log
TC_N=262144 timeout 300 python scripts/tc_c4_probe.py > gpurun_out/tc_plain2.log 2>&1 && \
TC_N=262144 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_dots -s 1 -c 1 -o gpurun_out/prof_tc -f python scripts/tc_c4_probe.py > gpurun_out/tc_ncu2.log 2>&1; echo "ncu2 rc=$?"

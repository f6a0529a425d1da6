mkdir -p gpurun_out
python scripts/tc_c4_probe.py > gpurun_out/tc_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv python scripts/tc_c4_probe.py > gpurun_out/tc_ncu1.log 2>&1; echo "ncu1 rc=$?"
cat gpurun_out/tc_plain.log
TC_N=262144 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_dots -s 1 -c 1 -o gpurun_out/prof_tc -f python scripts/tc_c4_probe.py > gpurun_out/tc_ncu2.log 2>&1; echo "ncu2 rc=$?"

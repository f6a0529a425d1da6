mkdir -p gpurun_out
TC_CFG=c3 TC_N=100000 TC_DATA=gauss TC_ITERS=6 python scripts/tc_breakdown.py > gpurun_out/c3_100k_plain.log 2>&1
TC_CFG=c3 TC_N=100000 TC_DATA=gauss TC_ITERS=6 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_100k.csv python scripts/tc_breakdown.py > /dev/null 2>&1
python scripts/launch_split.py gpurun_out/c3_100k.csv > gpurun_out/c3_100k_split.txt
SU_N=100000 true
cat gpurun_out/c3_100k_plain.log gpurun_out/c3_100k_split.txt

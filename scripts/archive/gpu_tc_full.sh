# One full ncu capture of the tensor-core filter sweep (tc_dots) at the C3
# and C4 shapes (column slices), plus the C2 bench line for regression.
mkdir -p gpurun_out
TC_CFG=c3 TC_N=524288 TC_ITERS=2 timeout 300 python scripts/tc_breakdown.py > gpurun_out/tcf_c3_plain.log 2>&1 && \
TC_CFG=c3 TC_N=524288 TC_ITERS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_dots -s 1 -c 1 -f -o gpurun_out/prof_tc_c3 python scripts/tc_breakdown.py > gpurun_out/tcf_c3.log 2>&1; echo "c3 rc=$?"
TC_CFG=c4 TC_N=262144 TC_ITERS=2 timeout 300 python scripts/tc_breakdown.py > gpurun_out/tcf_c4_plain.log 2>&1 && \
TC_CFG=c4 TC_N=262144 TC_ITERS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_dots -s 1 -c 1 -f -o gpurun_out/prof_tc_c4 python scripts/tc_breakdown.py > gpurun_out/tcf_c4.log 2>&1; echo "c4 rc=$?"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400

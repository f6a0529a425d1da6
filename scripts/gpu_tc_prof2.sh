# per-role cycle accounting of tc_dots (diagnostics build on the box)
GPSPCA_NVCC_FLAGS=-DGPS_TC_PROFILE python -m paper_1312_6182_b200._build > /dev/null
for m in ${MS:-16}; do for pr in ${PRS:-80}; do echo "m=$m probe=$pr"; TC_M=$m GPSPCA_TC_PROBE=$pr TC_INLINE=1 timeout 120 python scripts/tc_dots_probe.py 2>&1 | tail -14; done; done

# ncu --set full of tc_dots under GPSPCA_TC_PROBE variants (timing experiments)
mkdir -p gpurun_out
for pr in ${PROBES:-0 31}; do
  GPSPCA_TC_PROBE=$pr TC_N=262144 TC_INLINE=1 timeout 300 python scripts/tc_dots_probe.py > gpurun_out/tcp_$pr.log 2>&1 && \
  GPSPCA_TC_PROBE=$pr TC_N=262144 TC_INLINE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_dots -s 2 -c 1 \
     -o gpurun_out/prof_tc_p$pr -f python scripts/tc_dots_probe.py > gpurun_out/tcp_ncu_$pr.log 2>&1
  echo "probe $pr rc=$?"; cat gpurun_out/tcp_$pr.log
done

mkdir -p gpurun_out
python scripts/block_probe.py > gpurun_out/bp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bk_sweep -s 1 -c 1 -o gpurun_out/prof_bk -f python scripts/block_probe.py > gpurun_out/ncu_bk.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_bk.log

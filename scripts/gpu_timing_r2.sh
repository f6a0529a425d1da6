# Timing harness with both sides on the SAME box: the
# unmodified reference (baseline/_ref) on the host cores, then the device.
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/timing_ref_r2.log 2>&1
import sys, os
sys.path.insert(0, "baseline/_ref")
import gpspca
assert gpspca.__file__.startswith(os.path.abspath("baseline/_ref")), gpspca.__file__
cfg = gpspca.ExperimentConfig(timing_sizes=(500, 1000, 2000, 5000, 10000), timing_instances=3,
                              out="gpurun_out/timing_reference_cpu_r2.csv")
gpspca.run_timing_experiment(cfg)
print("reference done")
PY
echo "ref rc=$?"
python scripts/timing_device_run.py r2 > gpurun_out/timing_dev_r2.log 2>&1; echo "dev rc=$?"
python scripts/timing_compare.py gpurun_out/timing_reference_cpu_r2.csv gpurun_out/timing_device_r2.csv > gpurun_out/timing_r2_table.md
nproc >> gpurun_out/timing_r2_table.md

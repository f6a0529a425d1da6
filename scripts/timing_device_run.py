"""Device timing sweep on the paper's grid (P = N/10, m = 5, gamma in
{0.01, 0.05}, 3 instances per cell) -> profiles/timing_device_<tag>.csv."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1312_6182_b200 as gps  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
out = os.path.join("gpurun_out", f"timing_device_{tag}.csv")
cfg = gps.ExperimentConfig(timing_sizes=(500, 1000, 2000, 5000, 10000), timing_instances=3, device_columns=True,
                           out=out)
gps.run_timing_experiment(cfg)
print("wrote", out)

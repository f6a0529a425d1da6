#!/usr/bin/env python
"""Summarise the dense-activity ncu captures (scripts/gpu_round2_profiles.sh)
into profiles/ncu_dense_<tag>.json: per kernel the duration, DRAM bytes,
pipe utilisations (DMMA sub-pipe, FP64, XU), shared-memory wavefronts,
registers and occupancy.

    python scripts/summarize_dense.py <tag> <rep> [<rep> ...]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "dmma_pipe_pct_active": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct_active": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct_active": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct_active": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct_active": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "registers_per_thread": "launch__registers_per_thread",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    return [(dict(zip(h, r)), dict(zip(h, u))) for r in rows[2:]]


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    out = {"tag": tag, "kernels": []}
    for rep in reps:
        for d, units in raw(rep):
            k = {"capture": os.path.basename(rep), "kernel": d["Kernel Name"]}
            for name, metric in KEYS.items():
                v = d.get(metric, "")
                try:
                    val = float(v.replace(",", ""))
                except ValueError:
                    continue
                unit = units.get(metric, "")
                if unit == "Gbyte":
                    val *= 1e9
                elif unit == "Mbyte":
                    val *= 1e6
                elif unit == "usecond":
                    val /= 1e3
                elif unit == "nsecond":
                    val /= 1e6
                k[name] = val
            out["kernels"].append(k)
    path = os.path.join(ROOT, "profiles", f"ncu_dense_{tag}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

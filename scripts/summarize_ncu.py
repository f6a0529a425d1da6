#!/usr/bin/env python
"""Summarise gpurun_out/ ncu outputs into tracked files under profiles/.

    python scripts/summarize_ncu.py <launches.csv> <prof.ncu-rep> <tag> [p n]

writes profiles/ncu_launches_<tag>.txt (per-kernel launch list: count, mean
device time, share of the timed step) and profiles/ncu_sweep_<tag>.json
(--set full metrics of the sweep kernel: duration, DRAM bytes, throughput,
stall breakdown).  The newest sweep summary is also copied to
profiles/ncu_sweep_summary.json, which bench.py reads for `traffic`.
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[i], rows[i + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in data:
        if len(r) > vi and r[vi]:
            d[r[ki]].append(float(r[vi].replace(",", "")))
    return d


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    return [{n: (v, un) for n, un, v in zip(h, u, r)} for r in rows[2:]]


def main():
    lpath, rep, tag = sys.argv[1:4]
    p, n = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (4096, 1 << 20)
    d = launches(lpath)
    ours = {k: v for k, v in d.items() if "gps::" in k}
    step_total = sum(sum(v) / len(v) for k, v in ours.items() if any(s in k for s in ("sweep", "reduce", "step")))
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised); tag {tag}",
             f"# {'kernel':70s} {'launches':>8s} {'mean_us':>10s} {'share_of_iteration':>18s}"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        mean = sum(v) / len(v) / 1e3
        share = (sum(v) / len(v)) / step_total if k in ours and any(s in k for s in ("sweep", "reduce", "step")) else float("nan")
        lines.append(f"{k[:70]:70s} {len(v):8d} {mean:10.2f} {share:18.4f}")
    with open(os.path.join(ROOT, "profiles", f"ncu_launches_{tag}.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    rec = raw(rep)[0]
    g = lambda k: float(rec[k][0].replace(",", "")) if k in rec else None  # noqa: E731
    unit = lambda k: rec[k][1] if k in rec else None  # noqa: E731
    dur_ms = g("gpu__time_duration.sum") * (1e-6 if unit("gpu__time_duration.sum") == "ns" else
                                           1e-3 if unit("gpu__time_duration.sum") == "us" else 1.0)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = g("dram__bytes_read.sum") * scale[unit("dram__bytes_read.sum")]
    wr = g("dram__bytes_write.sum") * scale[unit("dram__bytes_write.sum")]
    stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: g(k) for k in rec
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1.0
    summary = {
        "tag": tag, "kernel": rec["Kernel Name"][0], "p": p, "n": n,
        "duration_ms": dur_ms, "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr, "algorithmic_bytes": p * n * 4,
        "traffic_over_algorithmic": (rd + wr) / (p * n * 4),
        "dram_GBps": (rd + wr) / (dur_ms * 1e-3) / 1e9,
        "registers_per_thread": g("launch__registers_per_thread"),
        "sm_throughput_pct": g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "dram_throughput_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "instructions": g("smsp__inst_executed.sum"),
        "stall_share": {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0)) if v},
    }
    for name in (f"ncu_sweep_{tag}.json", "ncu_sweep_summary.json"):
        with open(os.path.join(ROOT, "profiles", name), "w") as fh:
            json.dump(summary, fh, indent=1)
    print("\n".join(lines))
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()

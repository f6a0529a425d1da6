"""Compare the device timing sweep (paper_1312_6182_b200.timing) with the
reference CPU sweep CSV on the same (N, P = N/10) grid: per-cell median
seconds and iterations, and whether the iteration counts agree.

    python scripts/timing_compare.py profiles/timing_reference_cpu_r1.csv profiles/timing_device_r1.csv
"""
import csv
import sys
from collections import defaultdict


def load(path):
    med = {}
    per = defaultdict(dict)
    for r in csv.DictReader(open(path)):
        key = (r["variant"], int(r["N"]), float(r["gamma"]))
        if r["instance"] == "median":
            med[key] = (float(r["seconds"]), float(r["iterations"]))
        else:
            per[key][int(r["instance"])] = int(float(r["iterations"]))
    return med, per


def main(ref_path, dev_path):
    rmed, rper = load(ref_path)
    dmed, dper = load(dev_path)
    print("| variant | N | P | gamma | ref s (median) | device s (median) | speed-up | ref iters | device iters | iteration counts equal |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for key in sorted(set(rmed) & set(dmed), key=lambda k: (k[1], k[0], k[2])):
        v, N, g = key
        (rs, ri), (ds, di) = rmed[key], dmed[key]
        same = sum(rper[key].get(i) == dper[key].get(i) for i in rper[key])
        print(f"| {v} | {N} | {N // 10} | {g} | {rs:.4f} | {ds:.4f} | {rs / ds:.1f}x | {ri:g} | {di:g} | {same}/{len(rper[key])} |")


if __name__ == "__main__":
    main(*sys.argv[1:3])

"""Per-kernel time split of an ncu launch list (gpu__time_duration.sum CSV):
launches, mean and last duration per kernel name."""
import collections
import csv
import sys


def split(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    return agg


if __name__ == "__main__":
    for path in sys.argv[1:]:
        print(path)
        for k, v in split(path).items():
            if k.startswith("gps::") or "gps::" in k:
                print(f"  {k[:58]:58s} n={len(v):3d} mean={sum(v) / len(v):9.1f} us  last={v[-1]:9.1f} us")

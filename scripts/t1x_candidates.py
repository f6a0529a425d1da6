"""T1x workload at the bench's block configurations: the number of columns
T1 flags as candidates in the first sweep and how they fall on T1x's CTAs
(256-column items assigned round-robin over its grid), plus the per-iteration
time split.  Run twice: plainly (times) and with GPSPCA_TC_PROBE=512 (T1x
skipped, so T1's candidate mask survives for gpsdbg_bk_colmask).

    T1X_CFG=C3|C4|C4_dense python scripts/t1x_candidates.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_1312_6182_b200 as gps
    from paper_1312_6182_b200 import _native
    from paper_1312_6182_b200.block import BlockLoop, _top_m_columns

    want = os.environ.get("T1X_CFG", "C4")
    name, p, n, m, pen, mu, frac, data, k = [c for c in bench.BLOCK_CONFIGS if c[0] == want][0]
    dev = torch.device("cuda", 0)
    if data == "lowrank":
        n_classes, n_factors, support = (16, 10, n // 200) if name == "C3" else (32, 64, n // 128)
        At = bench.make_lowrank(torch, p, n, 0, n, dev, n_classes, n_factors, support)
    else:
        g = torch.Generator(device=dev)
        g.manual_seed(7)
        At = torch.randn((n, p), generator=g, device=dev, dtype=torch.float32)
    A = gps.DataMatrix.from_device(At.data_ptr(), p, n, owner=At, device=0)
    top = frac * float(A.norms.max())
    gamma = np.full(m, top if pen == "l1" else top * top)
    loop = BlockLoop(A, pen, m, gamma, mu, 0.0, 8)
    loop.start_columns(_top_m_columns(np.asarray(A.norms), m))
    L = _native.lib()
    probe = int(os.environ.get("GPSPCA_TC_PROBE", "0"))
    if probe & 512:
        _native.check(L.gps_bk_enqueue_sweep(loop.handle))
        mask = np.empty(2 * n, dtype=np.uint8)
        grid = _native.C.c_int()
        _native.check(L.gpsdbg_bk_colmask(loop.handle, mask.ctypes.data_as(_native._vp), _native.C.byref(grid)))
        cand = np.flatnonzero(mask[:n] | mask[n:])
        items = cand // 256
        per_cta = np.bincount(items % grid.value, minlength=grid.value)
        print(f"{name}: {cand.size} candidates in {np.unique(items).size} items; T1x grid {grid.value}; "
              f"per-CTA max {per_cta.max()}, CTAs with >16: {(per_cta > 16).sum()}, with 1..16: "
              f"{((per_cta > 0) & (per_cta <= 16)).sum()}; first columns {cand[:12].tolist()}")
        return
    s = torch.cuda.current_stream()
    for it in range(5):
        A.context.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        _native.check(L.gps_bk_enqueue_sweep(loop.handle))
        _native.check(L.gps_bk_enqueue_step(loop.handle))
        A.context.sync()
        e1.record(s)
        e1.synchronize()
        print(f"{name} iteration {it}: {e0.elapsed_time(e1):.3f} ms", flush=True)
    ns, ex = _native.C.c_int(), _native.C.c_int()
    if L.gpsdbg_bk_polar(loop.handle, _native.C.byref(ns), _native.C.byref(ex)) == 0:
        print(f"{name}: Newton-Schulz iterations {ns.value} over 5 polar steps, exact-path steps {ex.value}")


if __name__ == "__main__":
    main()

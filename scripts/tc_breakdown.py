"""Per-iteration time of the fp32 tensor-core block path (T0 split, T1 filter,
T1x exact recomputation, T2 update, K2 reduce, polar step) at the C3 / C4
shapes on Gaussian or planted low-rank+noise data, plus the active and
candidate-free column counts of the last sweep.  Run plainly for the
iteration times, and under `ncu --metrics gpu__time_duration.sum` for the
per-kernel split.

    TC_CFG=c3|c4  TC_DATA=gauss|planted  TC_DTYPE=f32|f64  TC_GFRAC=0.1  TC_ITERS=4 \
        python scripts/tc_breakdown.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def planted(torch, p, n, factors, support, seed):
    """SURVEY 8d C3/C4 distribution (reference datasets.py:278-309) built on
    the device: N(0, 1) noise plus rank-`factors` class structure on disjoint
    contiguous column supports."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    At = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float32)  # column-major p x n
    means = torch.randn((16, factors), generator=g, device="cuda") * 4.0
    latent = means[torch.arange(p, device="cuda") * 16 // p] + torch.randn((p, factors), generator=g, device="cuda")
    for f in range(factors):
        e = torch.randn(support, generator=g, device="cuda")
        e /= e.norm()
        At[f * support:(f + 1) * support, :] += e[:, None] * latent[:, f][None, :]
    return At


def main():
    import torch

    import paper_1312_6182_b200 as gps
    from paper_1312_6182_b200 import _native
    from paper_1312_6182_b200.block import BlockLoop, _top_m_columns

    cfg = os.environ.get("TC_CFG", "c3")
    data = os.environ.get("TC_DATA", "gauss")
    iters = int(os.environ.get("TC_ITERS", 4))
    if cfg == "c3":
        p, n, m, pen = 4096, int(os.environ.get("TC_N", 1 << 21)), 10, "l1"
        mu = np.ones(m)
        factors, support = 10, n // 200
    else:
        p, n, m, pen = 8192, int(os.environ.get("TC_N", 1 << 21)), 64, "l0"
        mu = np.linspace(1.0, 0.5, m)
        factors, support = 64, n // 128
    if data == "planted":
        At = planted(torch, p, n, factors, support, 3)
    else:
        g = torch.Generator(device="cuda")
        g.manual_seed(3)
        At = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float32)
    if os.environ.get("TC_DTYPE", "f32") == "f64":
        At = At.double()
        torch.cuda.empty_cache()
    A = gps.DataMatrix.from_device(At.data_ptr(), p, n, dtype=np.float64 if At.dtype == torch.float64 else np.float32,
                                   owner=At)
    top = float(os.environ.get("TC_GFRAC", 0.1)) * float(A.norms.max())
    gamma = np.full(m, top if pen == "l1" else top * top)
    loop = BlockLoop(A, pen, m, gamma, mu, 0.0, iters + 1)
    loop.start_columns(_top_m_columns(np.asarray(A.norms), m))
    L = _native.lib()
    s = torch.cuda.current_stream()
    times = []
    for it in range(iters):
        A.context.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        _native.check(L.gps_bk_enqueue_sweep(loop.handle))
        _native.check(L.gps_bk_enqueue_step(loop.handle))
        A.context.sync()
        e1.record(s)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        print(f"{cfg} {data} iteration {it}: {times[-1]:.3f} ms", flush=True)
    _native.check(L.gps_bk_run(loop.handle, 1))  # finishes the last iteration (max_iter reached)
    X, hist, conv, W, rf, rank = loop.result()
    active = int((W != 0).any(axis=1).sum())
    print(f"{cfg} {data} {A.dtype}: p={p} n={n} m={m} {pen}: median {np.median(times[1:] or times):.3f} ms/iteration, "
          f"active columns {active} ({100.0 * active / n:.2f}%), nnz {int((W != 0).sum())}, f={hist[-1]:.6g}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-config throughput sweep on one GPU.

Writes one JSON object per line to stdout and to profiles/configs_<tag>.jsonl:
iterations/s and A-stream GB/s of the device-resident power loop (fixed
iteration count, tol = 0), for the single-unit and block formulations at the
BASELINE shapes that fit one B200.  Data: Gaussian (the timing harness's
distribution, reference bench.py:245-246) generated on the device.

--cpu adds, per (formulation, n), the reference CPU path on the box's host
cores: real iterations of the unmodified reference (baseline/_ref) loop on
the same matrix (copied to the host) -- the whole matrix up to n = 2^20, a
2^20-column slice scaled linearly in n beyond (stated in the row).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gauss(torch, p, n, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.randn((n, p), generator=g, device="cuda", dtype=torch.float32)


def time_su(gps, torch, A, penalty, gamma, iters, warmup=3):
    from paper_1312_6182_b200 import _native

    loop = gps.single_unit.PowerLoop(A, penalty, gamma, 0.0, iters + warmup + 1)
    i = int(np.argmax(A.norms))
    loop.start(A.column(i) / A.norms[i])
    L = _native.lib()
    for _ in range(warmup):
        _native.check(L.gps_su_enqueue(loop.handle, 7))
    torch.cuda.synchronize()
    A.context.sync()
    t0 = time.perf_counter()
    for _ in range(iters):
        _native.check(L.gps_su_enqueue(loop.handle, 7))
    A.context.sync()
    return (time.perf_counter() - t0) / iters


def time_bk(gps, torch, A, penalty, m, gamma, mu, iters, warmup=2):
    from paper_1312_6182_b200 import _native
    from paper_1312_6182_b200.block import BlockLoop, _top_m_columns

    loop = BlockLoop(A, penalty, m, gamma, mu, 0.0, iters + warmup + 1)
    loop.start_columns(_top_m_columns(np.asarray(A.norms), m))
    L = _native.lib()
    for _ in range(warmup):
        _native.check(L.gps_bk_enqueue_sweep(loop.handle))
        _native.check(L.gps_bk_enqueue_step(loop.handle))
    A.context.sync()
    t0 = time.perf_counter()
    for _ in range(iters):
        _native.check(L.gps_bk_enqueue_sweep(loop.handle))
        _native.check(L.gps_bk_enqueue_step(loop.handle))
    A.context.sync()
    d, it, c = (_native.C.c_int() for _ in range(3))
    _native.check(L.gps_bk_poll(loop.handle, _native.C.byref(d), _native.C.byref(it), _native.C.byref(c)))
    assert not d.value, "block loop stopped early"
    return (time.perf_counter() - t0) / iters, full_reads(A, m)


def full_reads(A, m):
    """Full passes over A per block iteration: one for the tensor-core path
    (fp32, m >= 2: tc_dots reads A once; tc_refine / tc_update re-read only
    the candidate / active columns), else one per group of MG components."""
    if A.dtype == np.float32 and m >= 2:
        return 1
    mg = 4 if (A.dtype == np.float32 and A.p <= 4096) else 2
    return (m + mg - 1) // mg


CPU_MAX_COLS = 1 << 20


def ref_iteration_seconds(ref, A32, config, m, iters=1):
    """Seconds per iteration of the reference's own loop body on the host
    matrix A32 (p x cols fp32 view): single_unit.py:167-180 or
    block.py:211-224, best thread configuration of bench.py."""
    import bench
    from gpspca import block as rb

    A = ref.DataMatrix(A32)
    norms = ref.column_norms(A)
    top = float(norms.max())
    pen = "l1" if config[2] == "1" else "l0"
    gamma = 0.1 * top if pen == "l1" else (0.1 * top) ** 2
    _, workers, blas = bench.best_reference_config(ref, np.asarray(A32[:, : min(A32.shape[1], 65536)]),
                                                   os.cpu_count(), reps=1)
    if config.startswith("SL"):
        loop = bench.ReferenceLoop(ref, A, gamma, workers, blas)
        loop.first(A.column(int(np.argmax(norms))) / top)
        t0 = time.perf_counter()
        for _ in range(iters):
            loop.step()
        t = (time.perf_counter() - t0) / iters
        loop.close()
        return t, workers, blas
    from threadpoolctl import threadpool_limits

    plan = ref.KernelPlan(workers=workers, chunk=256)
    g = np.full(m, gamma)
    mu = np.ones(m)
    with threadpool_limits(blas, user_api="blas"):
        X = rb._init_block(A, ref.SolverConfig(penalty=pen, mode="block", m=m, gamma=gamma), plan)
        C = rb._correlations(A, X, plan)
        t0 = time.perf_counter()
        for _ in range(iters):
            G = rb._block_gradient(A, C, g, mu, pen, plan)
            X = rb.polar_projection(G).values
            C = rb._correlations(A, X, plan)
            rb._block_objective_from_correlations(C, g, mu, pen)
        t = (time.perf_counter() - t0) / iters
    return t, workers, blas


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--only", default="")
    ap.add_argument("--cpu", action="store_true", help="also time the reference CPU path (baseline/_ref)")
    args = ap.parse_args()
    ref = None
    if args.cpu:
        import bench

        ref = bench.import_reference()
    import torch

    import paper_1312_6182_b200 as gps

    out = []

    def emit(rec):
        print(json.dumps(rec), flush=True)
        out.append(rec)

    def cpu_rows(At, p, n):
        """The reference CPU path beside the device rows of this matrix."""
        cols = min(n, CPU_MAX_COLS)
        A32 = At[:cols].cpu().numpy().T
        for config, m in (("SL1", 1), ("SL0", 1), ("BL1 m=10", 10), ("BL0 m=10", 10)):
            t, workers, blas = ref_iteration_seconds(ref, A32, config, m)
            t_full = t * n / cols
            emit({"config": config, "p": p, "n": n, "impl": "reference-cpu", "iters_per_s": 1 / t_full,
                  "ms_per_iter": t_full * 1e3, "cores": os.cpu_count(), "workers": workers, "blas_threads": blas,
                  "sample": "whole matrix" if cols == n else f"first {cols} columns, scaled by n/{cols}"})

    def su_rows(p, n, seed, iters):
        At = gauss(torch, p, n, seed)
        if ref is not None:
            cpu_rows(At, p, n)
        A = gps.DataMatrix.from_device(At.data_ptr(), p, n, owner=At)
        del At
        top = float(A.norms.max())
        for pen, gamma in (("l1", 0.1 * top), ("l0", (0.1 * top) ** 2)):
            t = time_su(gps, torch, A, pen, gamma, iters)
            emit({"config": f"SL{pen[1]}", "p": p, "n": n, "iters_per_s": 1 / t, "ms_per_iter": t * 1e3,
                  "a_stream_gbs": p * n * 4 / t / 1e9, "reads_per_iter": 1})
        return A

    def bk_rows(A, m, iters, mu=None):
        top = float(A.norms.max())
        mu = np.ones(m) if mu is None else mu
        for pen, g in (("l1", 0.1 * top), ("l0", (0.1 * top) ** 2)):
            t, reads = time_bk(gps, torch, A, pen, m, np.full(m, g), mu, iters)
            emit({"config": f"BL{pen[1]} m={m}", "p": A.p, "n": A.n, "iters_per_s": 1 / t, "ms_per_iter": t * 1e3,
                  "reads_per_iter": reads, "a_stream_gbs": A.p * A.n * 4 * reads / t / 1e9})

    if args.only in ("", "c5"):
        for n in (100_000, 250_000, 500_000, 1 << 20, 1 << 21, 1 << 22, 1 << 23):
            A = su_rows(4096, n, n, 20 if n >= (1 << 21) else 50)
            bk_rows(A, 10, 5 if n >= (1 << 22) else 10)
            del A
            torch.cuda.empty_cache()
    if args.only in ("", "c4"):
        At = gauss(torch, 8192, 1 << 21, 4)
        A = gps.DataMatrix.from_device(At.data_ptr(), 8192, 1 << 21, owner=At)
        del At
        bk_rows(A, 64, 2, mu=np.linspace(1.0, 0.5, 64))
        del A
    with open(os.path.join(ROOT, "profiles", f"configs_{args.tag}.jsonl"), "w") as fh:
        for rec in out:
            fh.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()

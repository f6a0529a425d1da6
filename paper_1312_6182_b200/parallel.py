"""The reference's kernel seam (parallel.py:85-142), executed on the GPU.

Same names, argument meaning and errors as the reference.  `KernelPlan`
is accepted for signature compatibility: on the device the work split is a
fixed persistent grid (one CTA per SM, contiguous column stages) and the
cross-CTA reduction is a fixed-order sum, so results are bitwise
reproducible run to run for a given device, independent of `workers` --
the property the reference's pairwise tree buys on the CPU.
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import as_data_matrix

KERNELS = ("matvec_t", "gram_apply", "threshold_accumulate")


@dataclass(frozen=True)
class KernelPlan:
    """Execution plan (reference parallel.py:25-39); validated, then the
    device grid is chosen by the engine."""

    workers: int = 1
    chunk: int = 256
    reduction: str = "pairwise_tree"

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.chunk < 1:
            raise ValueError("chunk must be >= 1")
        if self.reduction != "pairwise_tree":
            raise ValueError("only the pairwise_tree reduction is supported")


DEFAULT_PLAN = KernelPlan()


def _vec(v, size, name):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.shape != (size,):
        raise ValueError(f"{name} must have length {size}, got shape {v.shape}")
    return v


def par_matvec_t(A, x, plan=DEFAULT_PLAN):
    """c = A'x, all column dot products (parallel.py:85-97)."""
    A = as_data_matrix(A)
    x = _vec(x, A.p, f"x (p={A.p})")
    out = np.empty(A.n)
    _native.check(_native.lib().gps_matvec_t(A.handle, _native.dptr(x), _native.dptr(out)))
    return out


def par_gram_apply(A, coefficients, plan=DEFAULT_PLAN):
    """sum_i c_i a_i = A c (parallel.py:108-114)."""
    A = as_data_matrix(A)
    c = _vec(coefficients, A.n, f"coefficients (n={A.n})")
    out = np.empty(A.p)
    _native.check(_native.lib().gps_gram_apply(A.handle, _native.dptr(c), _native.dptr(out)))
    return out


def threshold_weights(correlations, gamma, penalty):
    """w(c_i, gamma) on a host vector (parallel.py:117-128): l1 soft,
    l0 hard threshold with ties inactive.  The device kernels apply the
    same rule in registers (csrc/common.cuh threshold_weight)."""
    c = np.asarray(correlations, dtype=np.float64)
    if penalty == "l1":
        return np.sign(c) * np.maximum(np.abs(c) - gamma, 0.0)
    if penalty == "l0":
        return np.where(c * c > gamma, c, 0.0)
    raise ValueError(f"unknown penalty {penalty!r}")


def par_threshold_accumulate(A, correlations, gamma, penalty, plan=DEFAULT_PLAN):
    """sum_i w(c_i, gamma) a_i (parallel.py:131-142)."""
    A = as_data_matrix(A)
    c = _vec(correlations, A.n, f"correlations (n={A.n})")
    if penalty not in _native.PENALTY_CODE:
        raise ValueError(f"unknown penalty {penalty!r}")
    out = np.empty(A.p)
    _native.check(_native.lib().gps_threshold_accumulate(
        A.handle, _native.dptr(c), float(gamma), _native.PENALTY_CODE[penalty], _native.dptr(out)))
    return out


def fused_sweep(A, x, gamma, penalty, want_c=False, want_w=False):
    """One fused device sweep at x: (f, g/2, c or None, w or None, nnz).

    This is the engine's unit of work -- c = A'x, threshold, objective and
    the weighted column accumulation with a single read of A."""
    A = as_data_matrix(A)
    x = _vec(x, A.p, f"x (p={A.p})")
    if penalty not in _native.PENALTY_CODE:
        raise ValueError(f"unknown penalty {penalty!r}")
    f = _native.C.c_double(0.0)
    nnz = _native.C.c_int64(0)
    g = np.empty(A.p)
    c = np.empty(A.n) if want_c else None
    w = np.empty(A.n) if want_w else None
    _native.check(_native.lib().gps_su_sweep(
        A.handle, _native.dptr(x), float(gamma), _native.PENALTY_CODE[penalty], _native.C.byref(f),
        _native.dptr(g), _native.dptr(c) if want_c else None, _native.dptr(w) if want_w else None,
        _native.C.byref(nnz)))
    return f.value, g, c, w, nnz.value


def check_allocation(P, N, itemsize=8):
    """MemoryError before allocating a P x N matrix that cannot fit in the
    current device's free memory (the reference checks host RAM for its
    fp64 copy, parallel.py:145-157; the engine's copy lives in HBM)."""
    needed = int(P) * int(N) * int(itemsize)
    free = _native.C.c_size_t(0)
    if _native.lib().gps_device_free_bytes(_native.context().handle, _native.C.byref(free)) != _native.GPS_OK:
        return
    if needed > free.value:
        raise MemoryError(f"a {P}x{N} matrix needs {needed} bytes but only {free.value} are free on the device")


def _kernel_invocation(kernel, A, rng):
    if kernel == "matvec_t":
        x = rng.standard_normal(A.p)
        return lambda plan: par_matvec_t(A, x, plan)
    if kernel == "gram_apply":
        z = rng.standard_normal(A.n)
        return lambda plan: par_gram_apply(A, z, plan)
    if kernel == "threshold_accumulate":
        x = rng.standard_normal(A.p)
        c = par_matvec_t(A, x)
        gamma = 0.05 * float(np.max(np.abs(c)))
        return lambda plan: par_threshold_accumulate(A, c, gamma, "l1", plan)
    raise ValueError(f"unknown kernel {kernel!r}; expected one of {KERNELS}")


def measure_scaling(kernel, sizes, workers, instances=20, chunk=256, seed=0):
    """Median wall times of one kernel-seam call over a (P, N) grid and the
    given worker counts (parallel.py:175-215: same rows, order and
    speedup-vs-workers=1 definition).  On the device `workers` selects
    nothing -- the grid is fixed -- so the rows report the device call time
    per plan and speedups near 1; the harness is kept so callers of the
    reference's scaling table run unchanged."""
    import time

    if not sizes:
        raise ValueError("sizes must be nonempty")
    if instances < 1:
        raise ValueError("instances must be >= 1")
    if kernel not in KERNELS:
        raise ValueError(f"unknown kernel {kernel!r}; expected one of {KERNELS}")
    workers = sorted(set(int(w) for w in workers))
    if 1 not in workers:
        workers = [1] + workers
    rows = []
    for P, N in sorted(sizes, key=lambda s: s[1]):
        check_allocation(P, N)
        times = {w: [] for w in workers}
        for instance in range(instances):
            rng = np.random.default_rng([seed, N, instance])
            A = as_data_matrix(rng.standard_normal((P, N)))
            run = _kernel_invocation(kernel, A, rng)
            for w in workers:
                plan = KernelPlan(workers=w, chunk=chunk)
                start = time.perf_counter()
                run(plan)
                times[w].append(time.perf_counter() - start)
        base = float(np.median(times[1]))
        for w in workers:
            med = float(np.median(times[w]))
            rows.append({"kernel": kernel, "N": N, "P": P, "workers": w, "median_seconds": med,
                         "speedup": base / med if med > 0 else float("nan")})
    return rows

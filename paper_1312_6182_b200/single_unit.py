"""Single-unit sparse PCA (l1 / l0) on the GPU, mirroring reference
single_unit.py.

The power loop (`_iterate_single_unit`, reference single_unit.py:160-181)
runs entirely on the device: one fused sweep per iteration (K1) gives the
objective f_k and the next ascent direction in a single read of A, a
fixed-order reduction (K2) and the step kernel (K3) apply the stopping
rule and write x_{k+1} = g/||g|| and the history; the host launches
CUDA-graph chunks of iterations and polls the control block.  The loading
vector is read off the final sweep's thresholded correlations, so the
reference's extra recovery pass over A (single_unit.py:100-121) is free.

Sequential multi-component extraction keeps ONE device copy of A and
deflates implicitly (the step projects the gradient off the earlier
components) instead of materialising (I - xx')A per component.
"""

import os
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from .core import RunReport, SparseLoadings, as_data_matrix, decode_band, positive_part
from .parallel import DEFAULT_PLAN, fused_sweep, par_matvec_t

UNIT_NORM_TOL = 1e-9


def _poll_every():
    return max(1, int(os.environ.get("GPSPCA_POLL", "8")))


@dataclass(frozen=True)
class SingleUnitState:
    """Sphere iterate, its objective, and the step count (single_unit.py:26-32)."""

    x: np.ndarray
    objective: float
    iteration: int


def _check_unit(x, p):
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (p,):
        raise ValueError(f"x must have length p={p}, got shape {x.shape}")
    if abs(np.linalg.norm(x) - 1.0) > UNIT_NORM_TOL:
        raise ValueError("x must lie on the unit sphere")
    return x


def objective_sl1(A, x, gamma, plan=DEFAULT_PLAN):
    """sum_i [|a_i'x| - gamma]_+^2 (single_unit.py:51-56), one device sweep."""
    A = as_data_matrix(A)
    return fused_sweep(A, _check_unit(x, A.p), gamma, "l1")[0]


def objective_sl0(A, x, gamma, plan=DEFAULT_PLAN):
    """sum_i [(a_i'x)^2 - gamma]_+ (single_unit.py:59-64), one device sweep."""
    A = as_data_matrix(A)
    return fused_sweep(A, _check_unit(x, A.p), gamma, "l0")[0]


def _ascent(A, x, gamma, penalty):
    A = as_data_matrix(A)
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (A.p,):
        raise ValueError(f"x must have length p={A.p}, got shape {x.shape}")
    return 2.0 * fused_sweep(A, x, gamma, penalty)[1]


def ascent_direction_sl1(A, x, gamma, plan=DEFAULT_PLAN):
    """2 sum_i [|c_i| - gamma]_+ sign(c_i) a_i (single_unit.py:67-74)."""
    return _ascent(A, x, gamma, "l1")


def ascent_direction_sl0(A, x, gamma, plan=DEFAULT_PLAN):
    """2 sum_{c_i^2 > gamma} c_i a_i (single_unit.py:77-81)."""
    return _ascent(A, x, gamma, "l0")


def power_step(state, direction):
    """x+ = g/||g||, or a fixed point for g = 0 (single_unit.py:84-97)."""
    g = np.asarray(direction, dtype=np.float64)
    nrm = np.linalg.norm(g)
    if nrm == 0.0:
        return state, True
    return replace(state, x=g / nrm, iteration=state.iteration + 1), False


def _normalized(w):
    nrm = np.linalg.norm(w)
    return w / nrm if nrm > 0 else w


def _recover(A, x, gamma, penalty):
    A = as_data_matrix(A)
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (A.p,):
        raise ValueError(f"x must have length p={A.p}, got shape {x.shape}")
    return _normalized(fused_sweep(A, x, gamma, penalty, want_w=True)[3])


def recover_pattern_sl1(A, x, gamma, plan=DEFAULT_PLAN):
    """z = sign(c)[|c| - gamma]_+ / ||.|| at c = A'x (single_unit.py:100-111)."""
    return _recover(A, x, gamma, "l1")


def recover_pattern_sl0(A, x, gamma, plan=DEFAULT_PLAN):
    """z = c [c^2 > gamma] / ||.|| at c = A'x (single_unit.py:114-121)."""
    return _recover(A, x, gamma, "l0")


_RECOVER = {"l1": recover_pattern_sl1, "l0": recover_pattern_sl0}


class Trial(tuple):
    """(x, history, converged, w) of one loop run; `.band` holds the final
    sweep's near-threshold entries and their total count."""

    band = (np.zeros(0, dtype=np.int64), 0)


def _read_band(fn, handle, cap=8192):
    out = np.empty(cap, dtype=np.int64)
    cnt = _native.C.c_int(0)
    _native.check(fn(handle, out.ctypes.data_as(_native._i64p), cap, _native.C.byref(cnt)))
    return out[: min(cnt.value, cap)].copy(), int(cnt.value)


class PowerLoop:
    """Device power iteration for one (A, penalty, gamma, tol, max_iter):
    a gps_su object reused across restarts / components."""

    def __init__(self, A, penalty, gamma, tol, max_iter):
        self.A = A
        self.max_iter = int(max_iter)
        h = _native.C.c_void_p()
        _native.check(_native.lib().gps_su_create(
            A.handle, _native.PENALTY_CODE[penalty], float(gamma), float(tol), self.max_iter,
            _native.C.byref(h)), "gps_su_create")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            _native.lib().gps_su_destroy(h)
            self.handle = None

    def set_deflation(self, X):
        X = np.asfortranarray(X, dtype=np.float64) if X is not None and X.size else None
        k = 0 if X is None else X.shape[1]
        ptr = None if X is None else X.ctypes.data_as(_native._dp)
        _native.check(_native.lib().gps_su_set_deflation(self.handle, ptr, k))

    def start(self, x0):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        _native.check(_native.lib().gps_su_start(self.handle, _native.dptr(x0)))

    def run(self, x0, poll_every=None):
        """Iterate from x0 to the stopping rule; returns (x, history, converged, w)
        carrying the final sweep's near-threshold list as `.band`."""
        self.start(x0)
        _native.check(_native.lib().gps_su_run(self.handle, poll_every or _poll_every()), "power loop")
        trial = Trial(self.result())
        trial.band = self.band()
        return trial

    def band(self):
        """(entries, total) of the final sweep's near-threshold log."""
        return _read_band(_native.lib().gps_su_band, self.handle)

    def result(self):
        A = self.A
        x = np.empty(A.p)
        hist = np.empty(self.max_iter + 1)
        w = np.empty(A.n)
        nh = _native.C.c_int(0)
        conv = _native.C.c_int(0)
        s2 = _native.C.c_double(0.0)
        _native.check(_native.lib().gps_su_result(
            self.handle, _native.dptr(x), _native.dptr(hist), _native.C.byref(nh), _native.C.byref(conv),
            _native.dptr(w), _native.C.byref(s2)))
        return x, hist[: nh.value].tolist(), bool(conv.value), w


def _iterate_single_unit(A, x0, gamma, penalty, tol, max_iter, plan=DEFAULT_PLAN):
    """Power iteration from x0 (single_unit.py:160-181); (x, history, converged)."""
    A = as_data_matrix(A)
    x, history, converged, _ = PowerLoop(A, penalty, gamma, tol, max_iter).run(x0)
    return x, history, converged


def _activation_limit(norms, penalty):
    """single_unit.py:127-132: max_i ||a_i|| (l1) or its square (l0)."""
    top = float(np.max(norms))
    return top if penalty == "l1" else top * top


def _random_unit(rng, p):
    v = rng.standard_normal(p)
    return v / np.linalg.norm(v)


def _initial_iterates(A, config, norms=None, column=None):
    """Start directions (single_unit.py:135-157).  `norms` / `column` let the
    deflated path supply the norms and columns of (I - XX')A."""
    if config.init == "user_supplied":
        return [_check_unit(config.x0, A.p)]
    rng = np.random.default_rng(config.seed)
    if config.init == "random_orthonormal":
        return [_random_unit(rng, A.p) for _ in range(config.restarts)]
    norms = A.norms if norms is None else norms
    column = A.column if column is None else column
    order = np.argsort(-norms, kind="stable")[: config.restarts]
    out = [column(i) / norms[i] for i in order if norms[i] > 0]
    out += [_random_unit(rng, A.p) for _ in range(config.restarts - len(out))]
    return out


def _solve_component(A, gamma, config, plan=DEFAULT_PLAN, loop=None, norms=None, column=None, project=None,
                     info=None):
    """Shared single-component path (single_unit.py:267-284).

    Returns (z, history, converged, x).  `project` maps a start vector into
    the deflated space (implicit deflation).  `info` (a dict), if given,
    receives the final sweep's near-threshold list as info["band"]."""
    norms = A.norms if norms is None else norms
    if info is not None:
        info["band"] = Trial.band
    if gamma >= _activation_limit(norms, config.penalty):
        return np.zeros(A.n), [0.0], True, None
    loop = loop or PowerLoop(A, config.penalty, gamma, config.tol, config.max_iter)
    best = None
    for x0 in _initial_iterates(A, config, norms, column):
        trial = loop.run(project(x0) if project is not None else x0)
        if best is None or trial[1][-1] > best[1][-1]:
            best = trial
    if config.refine:
        from .refine import refine_support

        best = refine_support(A, best, gamma, config, loop, project=project)
    x, history, converged, w = best
    if info is not None:
        info["band"] = getattr(best, "band", Trial.band)
    return _normalized(w), history, converged, x


def solve_single_unit(A, config, plan=DEFAULT_PLAN):
    """One sparse component (single_unit.py:184-210) -> (SparseLoadings, RunReport)."""
    A = as_data_matrix(A)
    if config.mode != "single_unit":
        raise ValueError("solve_single_unit requires mode='single_unit'")
    if config.m != 1:
        raise ValueError("solve_single_unit handles m=1; use solve_multi_sequential")
    launches0 = A.context.launch_count
    start = time.perf_counter()
    info = {}
    z, history, converged, _ = _solve_component(A, float(config.gamma[0]), config, plan, info=info)
    band, band_total = info["band"]
    loadings = SparseLoadings(z)
    return loadings, RunReport(
        objective_history=history,
        iterations=len(history) - 1,
        wall_time=time.perf_counter() - start,
        nnz_per_component=loadings.nnz_per_component(),
        converged=converged,
        component_histories=[history],
        kernel_launches=A.context.launch_count - launches0,
        near_threshold=decode_band(band, 1),
        near_threshold_total=band_total,
    )


def deflate(A, x):
    """(I - xx')A as a new fp64 DataMatrix (single_unit.py:287-296).

    The solvers never call this (they deflate implicitly); it is kept for
    API parity and materialises the product on the device (x'A sweep, then
    a rank-1 update kernel writing the fp64 result)."""
    from .core import DataMatrix

    A = as_data_matrix(A)
    x = _check_unit(x, A.p)
    x = np.ascontiguousarray(x / np.linalg.norm(x))
    h = _native.C.c_void_p()
    _native.check(_native.lib().gps_matrix_deflate(A.handle, _native.dptr(x), _native.C.byref(h)))
    return DataMatrix._wrap(A.context, h)


class _ImplicitDeflation:
    """State of (I - XX')A for solve_multi_sequential: the orthonormal
    components X (p x j) and the correlations C = A'X (n x j) give the
    deflated column norms ||a_i||^2 - ||C_i||^2 and deflated columns
    a_i - X C_i without touching the device copy of A."""

    def __init__(self, A):
        self.A = A
        self.X = np.zeros((A.p, 0))
        self.C = np.zeros((A.n, 0))

    def add(self, x):
        x = _check_unit(x, self.A.p)
        x = x / np.linalg.norm(x)
        c = par_matvec_t(self.A, x)
        self.X = np.column_stack([self.X, x])
        self.C = np.column_stack([self.C, c])

    def norms(self):
        if self.X.shape[1] == 0:
            return self.A.norms
        sq = self.A.norms ** 2 - np.einsum("ij,ij->i", self.C, self.C)
        return np.sqrt(np.maximum(sq, 0.0))

    def column(self, i):
        a = self.A.column(i)
        for j in range(self.X.shape[1]):  # sequential projections, reference order
            a = a - self.X[:, j] * (self.X[:, j] @ a)
        return a

    def project(self, x):
        for j in range(self.X.shape[1]):
            x = x - self.X[:, j] * (self.X[:, j] @ x)
        return x


def _column_normed_norms(defl):
    """Deflated norms, re-evaluated exactly for the top candidates so the
    argmax / activation limit do not suffer from cancellation."""
    norms = np.array(defl.norms())
    if defl.X.shape[1]:
        top = np.argsort(-norms, kind="stable")[:8]
        for i in top:
            norms[i] = np.linalg.norm(defl.column(i))
    return norms


def solve_multi_sequential(A, config, plan=DEFAULT_PLAN):
    """config.m components by solve + deflate (single_unit.py:299-336)."""
    A = as_data_matrix(A)
    if config.mode != "single_unit":
        raise ValueError("solve_multi_sequential requires mode='single_unit'")
    launches0 = A.context.launch_count
    start = time.perf_counter()
    defl = _ImplicitDeflation(A)
    info = {}
    columns, histories, bands = [], [], []
    band_total = 0
    converged_all = True
    loops = {}
    for j in range(config.m):
        gamma = float(config.gamma[j])
        loop = loops.get(gamma)
        if loop is None:
            loop = loops[gamma] = PowerLoop(A, config.penalty, gamma, config.tol, config.max_iter)
        loop.set_deflation(defl.X)
        norms = _column_normed_norms(defl)
        z, history, converged, x = _solve_component(
            A, gamma, config, plan, loop=loop, norms=norms, column=defl.column,
            project=defl.project if defl.X.shape[1] else None, info=info)
        columns.append(z)
        histories.append(history)
        entries, total = info["band"]
        bands.append(decode_band(entries, 1)[0])
        band_total += total
        converged_all = converged_all and converged
        if not np.any(z):
            for _ in range(j + 1, config.m):
                columns.append(np.zeros(A.n))
                histories.append([0.0])
                bands.append(np.zeros(0, dtype=np.int64))
            break
        if j + 1 < config.m:
            defl.add(x)
    loadings = SparseLoadings(np.column_stack(columns))
    return loadings, RunReport(
        objective_history=histories[0],
        iterations=sum(len(h) - 1 for h in histories),
        wall_time=time.perf_counter() - start,
        nnz_per_component=loadings.nnz_per_component(),
        converged=converged_all,
        component_histories=histories,
        kernel_launches=A.context.launch_count - launches0,
        near_threshold=bands,
        near_threshold_total=band_total,
    )


__all__ = [
    "SingleUnitState", "objective_sl1", "objective_sl0", "ascent_direction_sl1", "ascent_direction_sl0",
    "power_step", "recover_pattern_sl1", "recover_pattern_sl0", "solve_single_unit", "deflate",
    "solve_multi_sequential", "positive_part",
]

"""Block sparse PCA (l1 / l0) on the Stiefel manifold, mirroring reference
block.py.

Each iteration runs ceil(m/MG) fused block sweeps (K1b: dots, per-component
mu scaling and threshold, objective, rank-MG update of the register-resident
G partial -- one read of A per group of MG components instead of the
reference's 2m reads) followed by the device polar step (Householder QR of
G, one-sided Jacobi SVD of R, X = Q U V'; block.py:135-149), with the
history and stopping rule on the device.  Initialisation is device
CholeskyQR2 (positive-diagonal R == the reference's sign-fixed QR).
"""

import os
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from .core import RunReport, SparseLoadings, StiefelPoint, as_data_matrix, decode_band
from .parallel import DEFAULT_PLAN, fused_sweep

BLOCK_FEASIBILITY_TOL = 1e-8  # block.py:17
_STATUS_STIEFEL = 3  # gps_bk loop status: an iterate missed the Stiefel tolerance


@dataclass(frozen=True)
class BlockState:
    """Stiefel iterate, objective, step count (block.py:20-30)."""

    X: StiefelPoint
    objective: float
    iteration: int


class RankDeficiencyError(RuntimeError):
    """Gradient lost full column rank (block.py:33-49); carries the rank,
    the requirement and, from the solve loop, the iteration index and the
    objective history up to the failure."""

    def __init__(self, rank, required, iteration=None):
        self.rank = rank
        self.required = required
        self.iteration = iteration
        where = "" if iteration is None else f" at iteration {iteration}"
        super().__init__(f"gradient has numerical rank {rank} < {required}{where}; reduce gamma or m")


def _as_stiefel_values(X, p, m=None):
    """block.py:52-63: shape check and ||X'X - I||_F <= 1e-8."""
    if isinstance(X, StiefelPoint):
        X = X.values
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    if X.shape[0] != p or (m is not None and X.shape[1] != m):
        raise ValueError(f"X must be {p}x{m or 'm'}, got {X.shape}")
    err = np.linalg.norm(X.T @ X - np.eye(X.shape[1]))
    if err > BLOCK_FEASIBILITY_TOL:
        raise ValueError(f"X is off the Stiefel manifold: ||X'X - I||_F = {err:.3e}")
    return X


def _per_component(vec, m, name):
    v = np.atleast_1d(np.asarray(vec, dtype=np.float64))
    if v.size == 1:
        v = np.full(m, v[0])
    if v.shape != (m,):
        raise ValueError(f"{name} must be a scalar or length-{m} vector")
    return np.ascontiguousarray(v)


def _fortran(X):
    return np.asfortranarray(X, dtype=np.float64)


def _block_sweep(A, X, gamma, mu, penalty, want_w=False):
    """One device block sweep: (f, G with the 2 mu_j factor, W or None)."""
    m = X.shape[1]
    Xf = _fortran(X)
    f = _native.C.c_double(0.0)
    G = np.empty((A.p, m), order="F")
    W = np.empty((A.n, m), order="F") if want_w else None
    _native.check(_native.lib().gps_bk_sweep(
        A.handle, Xf.ctypes.data_as(_native._dp), m, _native.dptr(gamma), _native.dptr(mu),
        _native.PENALTY_CODE[penalty], _native.C.byref(f), G.ctypes.data_as(_native._dp),
        W.ctypes.data_as(_native._dp) if want_w else None))
    return f.value, G, W


def _single_component_su(mu, gamma):
    return mu.size == 1 and mu[0] == 1.0


def objective_bl1(A, X, gamma, mu, plan=DEFAULT_PLAN):
    """sum_j sum_i [mu_j |a_i'x_j| - gamma_j]_+^2 (block.py:92-100)."""
    return _objective(A, X, gamma, mu, "l1")


def objective_bl0(A, X, gamma, mu, plan=DEFAULT_PLAN):
    """sum_j sum_i [(mu_j a_i'x_j)^2 - gamma_j]_+ (block.py:103-111)."""
    return _objective(A, X, gamma, mu, "l0")


def _objective(A, X, gamma, mu, penalty):
    A = as_data_matrix(A)
    X = _as_stiefel_values(X, A.p)
    m = X.shape[1]
    return _block_sweep(A, X, _per_component(gamma, m, "gamma"), _per_component(mu, m, "mu"), penalty)[0]


def ascent_direction_block(A, X, gamma, mu, penalty, plan=DEFAULT_PLAN):
    """G_j = 2 mu_j sum_i w(mu_j c_ij, gamma_j) a_i (block.py:124-132).  For
    m = 1 and mu = 1 this is the single-unit sweep, bitwise (test_block.py:115)."""
    A = as_data_matrix(A)
    X = _as_stiefel_values(X, A.p)
    m = X.shape[1]
    gamma = _per_component(gamma, m, "gamma")
    mu = _per_component(mu, m, "mu")
    if penalty not in _native.PENALTY_CODE:
        raise ValueError(f"unknown penalty {penalty!r}")
    if _single_component_su(mu, gamma):
        return (2.0 * fused_sweep(A, X[:, 0], float(gamma[0]), penalty)[1])[:, None]
    return _block_sweep(A, X, gamma, mu, penalty)[1]


def polar_projection(G):
    """Orthonormal polar factor U V' of G (block.py:135-149), on the device.
    Raises RankDeficiencyError(rank, m) when G is column-rank deficient by the
    reference rule s > s_0 max(p, m) eps."""
    G = np.asarray(G, dtype=np.float64)
    if G.ndim == 1:
        G = G[:, None]
    p, m = G.shape
    X = np.empty((p, m), order="F")
    rank = _native.C.c_int(0)
    ctx = _native.context()
    rc = _native.lib().gps_polar(ctx.handle, _fortran(G).ctypes.data_as(_native._dp), p, m,
                                 X.ctypes.data_as(_native._dp), _native.C.byref(rank))
    if rc == _native.GPS_E_RANK:
        raise RankDeficiencyError(rank.value, m)
    _native.check(rc, "polar_projection")
    return StiefelPoint(X)


def _polar_cholqr2(G):
    """polar_projection through the block loop's multi-CTA step (CholeskyQR2
    + Newton-Schulz with the Stiefel check and exact fallback, the path the
    loop takes for p m >= 4096): (X, ||X'X - I||_F, exact path taken)."""
    G = np.asarray(G, dtype=np.float64)
    p, m = G.shape
    X = np.empty((p, m), order="F")
    rank, exact = _native.C.c_int(0), _native.C.c_int(0)
    err = _native.C.c_double(0.0)
    rc = _native.lib().gps_polar_cholqr2(_native.context().handle, _fortran(G).ctypes.data_as(_native._dp), p, m,
                                         X.ctypes.data_as(_native._dp), _native.C.byref(rank), _native.C.byref(err),
                                         _native.C.byref(exact))
    if rc == _native.GPS_E_RANK:
        raise RankDeficiencyError(rank.value, m)
    _native.check(rc, "polar (CholeskyQR2 path)")
    return X, err.value, bool(exact.value)


class BlockLoop:
    """Device block power iteration (gps_bk) for one (A, penalty, m, gamma, mu)."""

    def __init__(self, A, penalty, m, gamma, mu, tol, max_iter):
        self.A, self.m, self.max_iter = A, int(m), int(max_iter)
        self.gamma = _per_component(gamma, m, "gamma")
        self.mu = _per_component(mu, m, "mu")
        h = _native.C.c_void_p()
        _native.check(_native.lib().gps_bk_create(
            A.handle, _native.PENALTY_CODE[penalty], self.m, _native.dptr(self.gamma), _native.dptr(self.mu),
            float(tol), self.max_iter, _native.C.byref(h)), "gps_bk_create")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            _native.lib().gps_bk_destroy(h)
            self.handle = None

    def start_user(self, X0):
        _native.check(_native.lib().gps_bk_start(self.handle, _fortran(X0).ctypes.data_as(_native._dp)))

    def start_qr(self, M):
        _native.check(_native.lib().gps_bk_start_qr(self.handle, _fortran(M).ctypes.data_as(_native._dp)))

    def start_columns(self, idx):
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        _native.check(_native.lib().gps_bk_start_columns(self.handle, idx.ctypes.data_as(_native._i64p)))

    def run(self, poll_every=8):
        _native.check(_native.lib().gps_bk_run(self.handle, poll_every), "block loop")
        X, history, converged, W, rank_fail, rank = self.result()
        stiefel, status, _ = self.diagnostics(len(history))
        self.stiefel_errors = stiefel
        if rank_fail:
            err = RankDeficiencyError(rank, self.m, iteration=len(history) - 1)
            err.history = history
            raise err
        if status == _STATUS_STIEFEL:  # the reference's StiefelPoint(U @ Vt) raises here (core.py:126-129)
            raise ValueError(f"columns not orthonormal: ||X'X - I||_F = {stiefel[-1]:.3e}")
        return X, history, converged, W

    def diagnostics(self, n_hist):
        """(per-iterate ||X'X - I||_F list, loop status, exact polar steps)."""
        out = np.zeros(n_hist + 1)
        status, exact = _native.C.c_int(0), _native.C.c_int(0)
        _native.check(_native.lib().gps_bk_diagnostics(self.handle, _native.dptr(out), _native.C.byref(status),
                                                       _native.C.byref(exact)))
        n = n_hist + (1 if status.value == _STATUS_STIEFEL else 0)
        return out[:n].tolist(), status.value, exact.value

    def band(self):
        """(entries, total) of the final sweep's near-threshold log."""
        from .single_unit import _read_band

        return _read_band(_native.lib().gps_bk_band, self.handle)

    def result(self):
        """(X, history, converged, W, rank_fail, rank) of the finished loop."""
        A, m = self.A, self.m
        X = np.empty((A.p, m), order="F")
        hist = np.empty(self.max_iter + 1)
        W = np.empty((A.n, m), order="F")
        nh, conv, rfail, rank = (_native.C.c_int(0) for _ in range(4))
        _native.check(_native.lib().gps_bk_result(
            self.handle, X.ctypes.data_as(_native._dp), _native.dptr(hist), _native.C.byref(nh),
            _native.C.byref(conv), W.ctypes.data_as(_native._dp), _native.C.byref(rfail), _native.C.byref(rank)))
        return X, hist[: nh.value].tolist(), bool(conv.value), W, bool(rfail.value), rank.value


def _top_m_columns(norms, m):
    """First m indices of argsort(-norms, kind='stable') (block.py:158)."""
    if m >= norms.size:
        return np.argsort(-norms, kind="stable")[:m]
    part = np.argpartition(-norms, m - 1)[:m]
    thr = norms[part].min()
    cand = np.flatnonzero(norms >= thr)
    order = cand[np.argsort(-norms[cand], kind="stable")]
    return order[:m]


def _recover_block(W):
    """block.py:174-187: Z_j = W_j / ||W_j|| (W already carries the mu scaling;
    the normalisation removes it)."""
    Z = np.zeros_like(W)
    for j in range(W.shape[1]):
        nrm = np.linalg.norm(W[:, j])
        if nrm > 0:
            Z[:, j] = W[:, j] / nrm
    return Z


def _init_x0(A, config, loop=None):
    """The initial iterate (block.py:152-171) on the device: with `loop`,
    written into the loop's X slot; without, returned as a host array."""
    p, m = A.p, config.m
    if config.init == "user_supplied":
        X0 = _as_stiefel_values(config.x0, p, m)
        StiefelPoint(X0)  # block.py:197 + core.py:118-129
        if loop is not None:
            loop.start_user(config.x0)
        return X0
    if config.init == "random_orthonormal":
        M = np.random.default_rng(config.seed).standard_normal((p, m))
    else:
        idx = _top_m_columns(np.asarray(A.norms), m)
        if loop is not None:
            loop.start_columns(idx)
            return None
        M = np.column_stack([A.column(i) for i in idx])
    if loop is not None:
        loop.start_qr(M)
        return None
    Q = np.empty((p, m), order="F")
    _native.check(_native.lib().gps_orthonormalize(_native.context().handle, _fortran(M).ctypes.data_as(_native._dp),
                                                   p, m, Q.ctypes.data_as(_native._dp)))
    return Q


def _eager_requested():
    """Trace mode: the module-level polar_projection was replaced (a caller
    intercepting every polar step, as the reference's acceptance criterion 5
    does, test_acceptance.py:195-228) or GPSPCA_EAGER_BLOCK=1."""
    import sys

    return (sys.modules[__name__].polar_projection is not _DEVICE_POLAR
            or os.environ.get("GPSPCA_EAGER_BLOCK") == "1")


def _solve_block_eager(A, config, start):
    """block.py:190-235 step by step from the host: one device block sweep
    per iteration (objective, G and W in one read of A) and a call of the
    module-level polar_projection (looked up at every step, so a
    replacement sees each G) -- the graph-captured loop's arithmetic,
    without the graph."""
    import sys

    mod = sys.modules[__name__]
    gamma, mu, m = config.gamma, config.mu, config.m
    point = StiefelPoint(_init_x0(A, config))
    stiefel = [float(np.linalg.norm(point.values.T @ point.values - np.eye(m)))]
    f, G, W = _block_sweep(A, point.values, gamma, mu, config.penalty, want_w=True)
    history = [f]
    converged = False
    iteration = 0
    while iteration < config.max_iter:
        try:
            point = mod.polar_projection(G)
        except RankDeficiencyError as err:
            err.iteration = iteration
            err.history = history
            raise
        X = point.values
        stiefel.append(float(np.linalg.norm(X.T @ X - np.eye(m))))
        f_new, G, W = _block_sweep(A, X, gamma, mu, config.penalty, want_w=True)
        history.append(f_new)
        iteration += 1
        if abs(f_new - f) < config.tol * max(abs(f), 1e-30):
            converged = True
            break
        f = f_new
    loadings = SparseLoadings(_recover_block(W))
    return loadings, RunReport(
        objective_history=history,
        iterations=len(history) - 1,
        wall_time=time.perf_counter() - start,
        nnz_per_component=loadings.nnz_per_component(),
        converged=converged,
        component_histories=[history],
        stiefel_errors=stiefel,
    )


def solve_block(A, config, plan=DEFAULT_PLAN, poll_every=8):
    """config.m components jointly (block.py:190-235) -> (SparseLoadings, RunReport)."""
    A = as_data_matrix(A)
    if config.mode != "block":
        raise ValueError("solve_block requires mode='block'")
    if not 1 <= config.m <= min(A.p, A.n):
        raise ValueError(f"need 1 <= m <= min(p, n) = {min(A.p, A.n)}, got m={config.m}")
    launches0 = A.context.launch_count
    start = time.perf_counter()
    if _eager_requested():
        loadings, report = _solve_block_eager(A, config, start)
        return loadings, replace(report, kernel_launches=A.context.launch_count - launches0)
    m = config.m
    loop = BlockLoop(A, config.penalty, m, config.gamma, config.mu, config.tol, config.max_iter)
    _init_x0(A, config, loop)
    X, history, converged, W = loop.run(poll_every)
    StiefelPoint(X)  # every polar output is a StiefelPoint in the reference (block.py:149, core.py:118-129)
    entries, total = loop.band()
    loadings = SparseLoadings(_recover_block(W))
    return loadings, RunReport(
        objective_history=history,
        iterations=len(history) - 1,
        wall_time=time.perf_counter() - start,
        nnz_per_component=loadings.nnz_per_component(),
        converged=converged,
        component_histories=[history],
        kernel_launches=A.context.launch_count - launches0,
        near_threshold=decode_band(entries, m),
        near_threshold_total=total,
        stiefel_errors=loop.stiefel_errors,
    )


_DEVICE_POLAR = polar_projection


__all__ = ["BlockState", "RankDeficiencyError", "objective_bl1", "objective_bl0", "ascent_direction_block",
           "polar_projection", "solve_block"]

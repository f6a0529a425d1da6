"""Column-chunked fp64 restatement of the reference loops for BASELINE-size
matrices -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference keeps an fp64 copy of A (core.py:36) and reads it twice per
single-unit iteration (single_unit.py:167-180: par_threshold_accumulate,
then par_matvec_t) and 2m times per block iteration (block.py:211-226).  At
the BASELINE sizes (C2 4096 x 2^20, C3 4096 x 2^21, C4 8192 x 2^21) that
copy is 34-137 GB, so this restatement keeps A in its fp32 storage and forms
fp64 products per column chunk: every chunk is widened to fp64 (exact) and
its dot products / weighted column sums are fp64 BLAS calls, exactly the
arithmetic the reference performs on those columns (parallel.py:85-142),
summed chunk by chunk in a fixed order (the reference's pairwise tree over
256-column chunks only moves the last bits).  The correlations of a sweep
and the gradient built from them come from ONE pass over the chunks (the
gradient uses the same correlations the reference's next step uses).
Chunks are processed by a thread pool (BLAS single-threaded per chunk).

Each function cites the reference lines it restates; thresholds, objective,
polar factor and initialisation reuse oracle.gpower.
"""

import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .gpower import EPS, OracleRankDeficiency, block_objective, polar, su_objective, threshold

__all__ = ["ChunkedA", "su_iterate_chunked", "block_solve_chunked"]


class ChunkedA:
    """A p x n fp32 (or fp64) Fortran-ordered host matrix swept in fp64 chunks."""

    def __init__(self, A, chunk=8192, workers=None):
        import os

        self.A = A
        self.p, self.n = A.shape
        self.chunk = chunk
        self.bounds = [(lo, min(lo + chunk, self.n)) for lo in range(0, self.n, chunk)]
        self.workers = workers or os.cpu_count()
        self._pool = ThreadPoolExecutor(self.workers)
        self._lock = threading.Lock()

    def _map(self, fn):
        from threadpoolctl import threadpool_limits

        with threadpool_limits(1, user_api="blas"):
            return list(self._pool.map(lambda b: fn(*b), self.bounds))

    def block(self, lo, hi):
        return np.asarray(self.A[:, lo:hi], dtype=np.float64)

    def column(self, i):
        return np.asarray(self.A[:, i], dtype=np.float64)

    def norms(self):
        """core.py:243-246 -- fp64 column norms."""
        out = np.empty(self.n)

        def f(lo, hi):
            out[lo:hi] = np.linalg.norm(self.block(lo, hi), axis=0)

        self._map(f)
        return out

    def sweep(self, X, gamma, mu, penalty):
        """One pass: C = A'X (parallel.py:85-97 per column), then
        G_j = sum_i w(mu_j c_ij, gamma_j) a_i (parallel.py:131-142,
        block.py:114-121 without the 2 mu_j factor).  Returns (C, G)."""
        X = np.asarray(X, dtype=np.float64)
        if X.ndim == 1:
            X = X[:, None]
        m = X.shape[1]
        gamma = np.broadcast_to(np.asarray(gamma, dtype=np.float64), (m,))
        mu = np.broadcast_to(np.asarray(mu, dtype=np.float64), (m,))
        C = np.empty((self.n, m))

        def f(lo, hi):
            B = self.block(lo, hi)
            Cb = B.T @ X
            C[lo:hi] = Cb
            W = np.column_stack([threshold(mu[j] * Cb[:, j], gamma[j], penalty) for j in range(m)])
            return B @ W

        parts = self._map(f)
        G = np.zeros((self.p, m))
        for part in parts:  # fixed chunk order
            G += part
        return C, G


def su_iterate_chunked(A, x0, gamma, penalty, tol, max_iter):
    """single_unit.py:160-181 on a ChunkedA; returns (x, history, converged, c_final)."""
    x = np.asarray(x0, dtype=np.float64)
    c, g = A.sweep(x, gamma, 1.0, penalty)
    c = c[:, 0]
    f = su_objective(c, gamma, penalty)
    history = [f]
    converged = False
    for _ in range(max_iter):
        g = 2.0 * g[:, 0]
        nrm = np.linalg.norm(g)
        if nrm == 0.0:
            converged = True
            break
        x = g / nrm
        c, g = A.sweep(x, gamma, 1.0, penalty)
        c = c[:, 0]
        f_new = su_objective(c, gamma, penalty)
        history.append(f_new)
        if abs(f_new - f) < tol * max(abs(f), 1e-30):
            converged = True
            break
        f = f_new
    return x, history, converged, c


def block_solve_chunked(A, m, gamma, mu, penalty, tol, max_iter, X0):
    """block.py:190-235 on a ChunkedA from a given X0 (block.py:202-226):
    returns (C_final, history, converged, X_final); rank loss raises
    OracleRankDeficiency with .iteration / .history (block.py:215-218)."""
    gamma = np.broadcast_to(np.asarray(gamma, dtype=np.float64), (m,)).copy()
    mu = np.broadcast_to(np.asarray(mu, dtype=np.float64), (m,)).copy()
    X = np.asarray(X0, dtype=np.float64)
    C, Gh = A.sweep(X, gamma, mu, penalty)
    f = block_objective(C, gamma, mu, penalty)
    history = [f]
    converged = False
    it = 0
    while it < max_iter:
        G = Gh * (2.0 * mu)[None, :]
        try:
            X = polar(G)
        except OracleRankDeficiency as err:
            err.iteration, err.history = it, history
            raise
        C, Gh = A.sweep(X, gamma, mu, penalty)
        f_new = block_objective(C, gamma, mu, penalty)
        history.append(f_new)
        it += 1
        if abs(f_new - f) < tol * max(abs(f), 1e-30):
            converged = True
            break
        f = f_new
    return C, history, converged, X


def max_norm_start(A, m, norms=None):
    """block.py:152-170 max_norm_column init (and single_unit.py:151-156
    for m = 1 without the QR): QR of the top-m columns, sign-fixed."""
    norms = A.norms() if norms is None else norms
    idx = np.argsort(-norms, kind="stable")[:m]
    M = np.column_stack([A.column(i) for i in idx])
    Q, R = np.linalg.qr(M)
    d = np.diagonal(R)
    if np.any(np.abs(d) <= m * EPS * max(1.0, np.abs(d).max())):
        raise ValueError("initialization columns are numerically rank deficient")
    return Q * np.sign(d), idx

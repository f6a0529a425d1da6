"""NumPy fp64 restatement of the reference GP-SPCA power iteration.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites
the reference file:line it restates; paths are relative to
`/root/reference/pkg/src/gpspca/`.  The restatement is deliberately plain
(whole-matrix BLAS calls, no chunking or thread pool): the reference's
chunked pairwise-tree summation order (parallel.py:74-82) only moves the
last bits, which the parity tolerances absorb.

Arguments follow the reference conventions: A is p x n (columns are the
variables), x lives in R^p, c = A'x in R^n, loadings z in R^n.
"""

import numpy as np

__all__ = [
    "OracleRankDeficiency",
    "column_norms",
    "threshold",
    "su_objective",
    "su_gradient",
    "su_iterate",
    "su_initial_points",
    "su_solve",
    "su_recover",
    "deflate",
    "multi_sequential",
    "block_correlations",
    "block_objective",
    "block_gradient",
    "polar",
    "block_initial_point",
    "block_recover",
    "block_solve",
    "activation_limit",
]

EPS = np.finfo(np.float64).eps


class OracleRankDeficiency(RuntimeError):
    """Mirror of block.py:33-49 RankDeficiencyError (rank, required, iteration)."""

    def __init__(self, rank, required, iteration=None, history=None):
        super().__init__(f"rank {rank} < {required} (iteration {iteration})")
        self.rank, self.required, self.iteration, self.history = rank, required, iteration, history


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def column_norms(A):
    """core.py:243-246 -- Euclidean norm of every column."""
    return np.linalg.norm(_f64(A), axis=0)


def threshold(c, gamma, penalty):
    """parallel.py:117-128 -- l1 soft threshold sign(c)(|c|-g)_+ ; l0 hard
    threshold c*[c^2 > g] (a tie c^2 == g is inactive)."""
    c = _f64(c)
    if penalty == "l1":
        return np.sign(c) * np.maximum(np.abs(c) - gamma, 0.0)
    if penalty == "l0":
        return np.where(c * c > gamma, c, 0.0)
    raise ValueError(penalty)


def su_objective(c, gamma, penalty):
    """single_unit.py:44-48 -- sum (|c|-g)_+^2 (l1) or sum (c^2-g)_+ (l0)."""
    c = _f64(c)
    if penalty == "l1":
        t = np.maximum(np.abs(c) - gamma, 0.0)
        return float(np.dot(t, t))
    return float(np.maximum(c * c - gamma, 0.0).sum())


def su_gradient(A, c, gamma, penalty):
    """single_unit.py:168 / parallel.py:131-142 -- 2 * sum_i w(c_i) a_i."""
    return 2.0 * (_f64(A) @ threshold(c, gamma, penalty))


def activation_limit(norms, penalty):
    """single_unit.py:127-132 -- largest gamma at which a column can activate."""
    top = float(np.max(norms))
    return top if penalty == "l1" else top * top


def su_iterate(A, x0, gamma, penalty, tol, max_iter):
    """single_unit.py:160-181 -- the power loop; returns (x, history, converged)."""
    A = _f64(A)
    x = _f64(x0)
    c = A.T @ x
    f = su_objective(c, gamma, penalty)
    history = [f]
    converged = False
    for _ in range(max_iter):
        g = su_gradient(A, c, gamma, penalty)
        nrm = np.linalg.norm(g)
        if nrm == 0.0:
            converged = True
            break
        x = g / nrm
        c = A.T @ x
        f_new = su_objective(c, gamma, penalty)
        history.append(f_new)
        if abs(f_new - f) < tol * max(abs(f), 1e-30):
            converged = True
            break
        f = f_new
    return x, history, converged


def _unit_checked(x, p):
    """single_unit.py:35-41 -- shape (p,) and | ||x|| - 1 | <= 1e-9."""
    x = _f64(x)
    if x.shape != (p,) or abs(np.linalg.norm(x) - 1.0) > 1e-9:
        raise ValueError("x must be a unit vector of length p")
    return x


def su_initial_points(A, init="max_norm_column", seed=0, restarts=1, x0=None):
    """single_unit.py:135-157 -- start directions for each restart."""
    A = _f64(A)
    p = A.shape[0]
    if init == "user_supplied":
        return [_unit_checked(x0, p)]
    rng = np.random.default_rng(seed)

    def _rand():
        v = rng.standard_normal(p)
        return v / np.linalg.norm(v)

    if init == "random_orthonormal":
        return [_rand() for _ in range(restarts)]
    norms = column_norms(A)
    picks = np.argsort(-norms, kind="stable")[:restarts]
    starts = [A[:, i] / norms[i] for i in picks if norms[i] > 0]
    starts += [_rand() for _ in range(restarts - len(starts))]
    return starts


def su_recover(A, x, gamma, penalty):
    """single_unit.py:100-121 -- z = w(A'x)/||w(A'x)|| (zero stays zero)."""
    z = threshold(_f64(A).T @ _f64(x), gamma, penalty)
    nrm = np.linalg.norm(z)
    return z / nrm if nrm > 0 else z


def su_solve(A, gamma, penalty="l1", tol=1e-6, max_iter=1000, init="max_norm_column",
             seed=0, restarts=1, x0=None):
    """single_unit.py:267-284 (_solve_component, refine=False).

    Returns (z, history, converged, x) with x None when gamma is past the
    activation limit.
    """
    A = _f64(A)
    if gamma >= activation_limit(column_norms(A), penalty):
        return np.zeros(A.shape[1]), [0.0], True, None
    best = None
    for start in su_initial_points(A, init, seed, restarts, x0):
        trial = su_iterate(A, start, gamma, penalty, tol, max_iter)
        if best is None or trial[1][-1] > best[1][-1]:
            best = trial
    x, history, converged = best
    return su_recover(A, x, gamma, penalty), history, converged, x


def deflate(A, x):
    """single_unit.py:287-296 -- (I - xx')A with x renormalized."""
    A = _f64(A)
    x = _unit_checked(x, A.shape[0])
    x = x / np.linalg.norm(x)
    return A - np.outer(x, x @ A)


def multi_sequential(A, gammas, penalty="l1", tol=1e-6, max_iter=1000,
                     init="max_norm_column", seed=0, restarts=1, x0=None):
    """single_unit.py:299-336 -- m components by solve + deflate.

    Returns (Z n x m, histories, converged_all).
    """
    A = _f64(A)
    m = len(gammas)
    cols, histories, conv_all = [], [], True
    current = A
    for j in range(m):
        z, hist, conv, x = su_solve(current, float(gammas[j]), penalty, tol, max_iter,
                                    init, seed, restarts, x0)
        cols.append(z)
        histories.append(hist)
        conv_all = conv_all and conv
        if not np.any(z):
            for _ in range(j + 1, m):
                cols.append(np.zeros(A.shape[1]))
                histories.append([0.0])
            break
        if j + 1 < m:
            current = deflate(current, x)
    return np.column_stack(cols), histories, conv_all


# ----------------------------------------------------------------- block


def block_correlations(A, X):
    """block.py:75-77 -- C = A'X (n x m)."""
    return _f64(A).T @ _f64(X)


def block_objective(C, gamma, mu, penalty):
    """block.py:80-89 -- sum_j sum_i [mu_j|c_ij| - g_j]_+^2 or [(mu_j c_ij)^2 - g_j]_+."""
    S = _f64(C) * _f64(mu)[None, :]
    g = _f64(gamma)[None, :]
    if penalty == "l1":
        t = np.maximum(np.abs(S) - g, 0.0)
        return float(sum(np.dot(t[:, j], t[:, j]) for j in range(S.shape[1])))
    return float(sum(np.maximum(S[:, j] ** 2 - g[0, j], 0.0).sum() for j in range(S.shape[1])))


def block_gradient(A, C, gamma, mu, penalty):
    """block.py:114-121 -- G_j = 2 mu_j sum_i w(mu_j c_ij, g_j) a_i."""
    A = _f64(A)
    mu = _f64(mu)
    gamma = _f64(gamma)
    W = np.column_stack([threshold(mu[j] * C[:, j], gamma[j], penalty) for j in range(C.shape[1])])
    return (A @ W) * (2.0 * mu)[None, :]


def polar(G):
    """block.py:135-149 -- U V' from the thin SVD, with the reference rank rule
    (s > s0 * max(p, m) * eps, rank 0 when s0 == 0)."""
    G = _f64(G)
    if G.ndim == 1:
        G = G[:, None]
    U, s, Vt = np.linalg.svd(G, full_matrices=False)
    cutoff = s[0] * max(G.shape) * EPS
    rank = int(np.count_nonzero(s > cutoff)) if s[0] > 0 else 0
    if rank < G.shape[1]:
        raise OracleRankDeficiency(rank, G.shape[1])
    return U @ Vt


def block_initial_point(A, m, init="max_norm_column", seed=0, X0=None):
    """block.py:152-171 -- QR of the top-m-norm columns (or Gaussian) with the
    sign of diag(R) folded into Q; user_supplied is returned as is."""
    A = _f64(A)
    p = A.shape[0]
    if init == "user_supplied":
        X0 = _f64(X0).reshape(p, m)
        if np.linalg.norm(X0.T @ X0 - np.eye(m)) > 1e-8:
            raise ValueError("X0 off the Stiefel manifold")
        return X0
    if init == "random_orthonormal":
        M = np.random.default_rng(seed).standard_normal((p, m))
    else:
        M = A[:, np.argsort(-column_norms(A), kind="stable")[:m]].copy()
    Q, R = np.linalg.qr(M)
    d = np.diagonal(R)
    if np.any(np.abs(d) <= m * EPS * max(1.0, np.abs(d).max())):
        raise ValueError("initialization columns are numerically rank deficient")
    return Q * np.sign(d)


def block_recover(C, gamma, mu, penalty):
    """block.py:174-187 -- Z_j from the final correlations, unit-normalized."""
    n, m = C.shape
    Z = np.zeros((n, m))
    for j in range(m):
        c = C[:, j]
        if penalty == "l1":
            v = np.sign(c) * np.maximum(mu[j] * np.abs(c) - gamma[j], 0.0)
        else:
            s = mu[j] * c
            v = np.where(s * s > gamma[j], c, 0.0)
        nrm = np.linalg.norm(v)
        if nrm > 0:
            Z[:, j] = v / nrm
    return Z


def block_solve(A, m, gamma, mu=1.0, penalty="l1", tol=1e-6, max_iter=1000,
                init="max_norm_column", seed=0, X0=None):
    """block.py:190-235 -- returns (Z, history, converged, X).

    Raises OracleRankDeficiency with .iteration/.history on gradient rank loss.
    """
    A = _f64(A)
    gamma = np.broadcast_to(_f64(gamma), (m,)).copy()
    mu = np.broadcast_to(_f64(mu), (m,)).copy()
    X = block_initial_point(A, m, init, seed, X0)
    C = block_correlations(A, X)
    f = block_objective(C, gamma, mu, penalty)
    history = [f]
    converged = False
    it = 0
    while it < max_iter:
        G = block_gradient(A, C, gamma, mu, penalty)
        try:
            X = polar(G)
        except OracleRankDeficiency as err:
            err.iteration, err.history = it, history
            raise
        C = block_correlations(A, X)
        f_new = block_objective(C, gamma, mu, penalty)
        history.append(f_new)
        it += 1
        if abs(f_new - f) < tol * max(abs(f), 1e-30):
            converged = True
            break
        f = f_new
    return block_recover(C, gamma, mu, penalty), history, converged, X

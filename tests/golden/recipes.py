"""Input recipes shared by the golden generator and the tests (no reference
import here: this module travels to the GPU box)."""

import hashlib

import numpy as np


def make_matrix(recipe):
    """Rebuild A from a recipe dict (mirrored in tests/golden_util.py)."""
    kind = recipe["kind"]
    p, n = recipe["shape"]
    if kind == "gauss32":
        A = np.random.default_rng(recipe["seed"]).standard_normal((p, n)).astype(np.float32)
    elif kind == "lowrank32":
        rng = np.random.default_rng(recipe["seed"])
        k = recipe["rank"]
        U = rng.standard_normal((p, k))
        V = np.zeros((n, k))
        s = recipe["support"]
        for f in range(k):
            e = rng.standard_normal(s)
            V[f * s:(f + 1) * s, f] = e / np.linalg.norm(e)
        A = (U * recipe["scale"]) @ V.T + rng.standard_normal((p, n))
        A = A.astype(np.float32)
    elif kind == "nearcol":
        # Gaussian with the two largest columns nearly (or exactly) collinear:
        # a_0 scaled up, a_1 = a_0 + rel * ||a_0|| * e (built in fp64, so
        # the matrix must be stored as fp64 to keep the perturbation)
        rng = np.random.default_rng(recipe["seed"])
        A = rng.standard_normal((p, n)).astype(np.float32).astype(np.float64)
        A[:, 0] *= 10.0
        e = rng.standard_normal(p)
        A[:, 1] = A[:, 0] + recipe["rel"] * np.linalg.norm(A[:, 0]) * e / np.linalg.norm(e)
        return A
    elif kind == "zeros":
        A = np.zeros((p, n), dtype=np.float32)
    elif kind == "diag":
        A = np.zeros((p, n), dtype=np.float32)
        d = recipe["diag"]
        for i, v in enumerate(d):
            A[i, i] = v
    else:
        raise ValueError(kind)
    return A.astype(np.float64)


def digest(A):
    return hashlib.sha256(np.asfortranarray(A).tobytes()).hexdigest()[:16]


def polar_input(recipe):
    """G = U diag(s) V' with Haar-like U (p x m), V (m x m): s is
    logspace(0, -log10 kappa, m) or an explicit list."""
    rng = np.random.default_rng(recipe["seed"])
    p, m = recipe["p"], recipe["m"]
    U = np.linalg.qr(rng.standard_normal((p, m)))[0]
    V = np.linalg.qr(rng.standard_normal((m, m)))[0]
    s = np.asarray(recipe["s"], dtype=np.float64) if "s" in recipe else np.logspace(0, -np.log10(recipe["kappa"]), m)
    return (U * s) @ V.T


# ---- recognition-path fixtures (make_golden_recog.py) ----

def recog_samples(seed, n, f):
    rng = np.random.default_rng(seed)
    base = rng.standard_normal((n, 3)) @ rng.standard_normal((3, f)) * 2.0
    return (base + rng.standard_normal((n, f))).astype(np.float32).astype(np.float64)


def sparse_loadings(seed, f, m, nnz):
    rng = np.random.default_rng(seed)
    L = np.zeros((f, m))
    for j in range(m):
        idx = rng.choice(f, size=nnz, replace=False)
        L[idx, j] = rng.standard_normal(nnz)
        L[:, j] /= np.linalg.norm(L[:, j])
    L[:, -1] = 0.0  # a zero component (explained_variance credits 0)
    return L


def knn_case(seed, r, t, dim, n_labels, dup):
    rng = np.random.default_rng(seed)
    train = rng.standard_normal((r, dim))
    test = rng.standard_normal((t, dim))
    if dup:  # exact ties: repeated train rows and test rows on train rows
        train[5] = train[2]
        train[r - 1] = train[2]
        test[0] = train[2]
        test[1] = train[r // 2 + 1]
    labels = rng.integers(0, n_labels, size=r)
    return train, labels, test

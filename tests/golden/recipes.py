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

"""Oracle for the recognition path -- TEST INFRASTRUCTURE
ONLY.  NumPy fp64 restatements of the reference's projection, explained
variance, k-NN and dense PCA, each citing the reference lines it follows
(`/root/reference/pkg/src/gpspca/`).  Pinned by tests/golden/recog.json,
which tests/golden/make_golden_recog.py produced by running the reference.
"""

import numpy as np

__all__ = ["sign_fix", "dense_pca", "embed", "variance_explained", "knn_predict"]


def sign_fix(L):
    """pca.py:25-34: each column's largest-|.| entry made positive (first
    such entry on ties, as np.argmax)."""
    L = np.array(L, dtype=np.float64)
    idx = np.argmax(np.abs(L), axis=0)
    flip = L[idx, np.arange(L.shape[1])] < 0
    L[:, flip] *= -1.0
    return L


def dense_pca(S, m):
    """pca.py:37-54: leading right singular vectors of the centred samples."""
    S = np.asarray(S, dtype=np.float64)
    mu = S.mean(axis=0)
    _, sv, vt = np.linalg.svd(S - mu, full_matrices=False)
    return sign_fix(vt[:m].T), sv[:m].copy(), mu


def embed(S, L, mean=None):
    """pca.py:57-71: (S - mean) L, mean defaulting to S's column means."""
    S = np.asarray(S, dtype=np.float64)
    L = np.asarray(L, dtype=np.float64)
    mu = S.mean(axis=0) if mean is None else np.asarray(mean, dtype=np.float64)
    return (S - mu) @ L


def variance_explained(S, L, zero_tol=1e-12):
    """pca.py:74-103: per-component variance of the centred data after
    projecting out the earlier (nonzero) components one by one."""
    S = np.asarray(S, dtype=np.float64)
    L = np.asarray(L, dtype=np.float64)
    if L.ndim == 1:
        L = L[:, None]
    keep = np.linalg.norm(L, axis=0) > zero_tol
    B = S - S.mean(axis=0)
    den = max(S.shape[0] - 1, 1)
    out = np.zeros(L.shape[1])
    for j in np.nonzero(keep)[0]:
        sc = B @ L[:, j]
        out[j] = float(sc @ sc) / den
        B = B - np.outer(sc, L[:, j])
    return out


def knn_predict(train, train_labels, test, k=1):
    """datasets.py:213-270: squared distances by (|t|^2 - 2 t.s) + |s|^2
    clamped at 0; k = 1 takes the first minimum; k > 1 the stable-sorted
    first k, majority label, ties to the label of the nearest tied
    neighbour."""
    train = np.asarray(train, dtype=np.float64)
    test = np.asarray(test, dtype=np.float64)
    labels = np.asarray(train_labels)
    d = (np.sum(test * test, axis=1)[:, None] - 2.0 * test @ train.T) + np.sum(train * train, axis=1)[None, :]
    d = np.maximum(d, 0.0)
    if k == 1:
        return labels[np.argmin(d, axis=1)]
    out = np.empty(test.shape[0], dtype=labels.dtype)
    nearest = np.argsort(d, axis=1, kind="stable")[:, :k]
    for r, row in enumerate(nearest):
        votes = labels[row]
        uniq, cnt = np.unique(votes, return_counts=True)
        best = uniq[cnt == cnt.max()]
        out[r] = best[0] if best.size == 1 else next(labels[i] for i in row if labels[i] in best)
    return out

"""Recognition path on the device: projection,
explained variance, k-NN classification and the dense PCA baseline.

Same names, arguments and errors as the reference (`pca.py:16-103`,
`datasets.py:213-275`).  The arithmetic runs in libgpspca_b200:

* `project` / `explained_variance`: Y = S L in one pass over the columns
  (features) with a nonzero loading (`gps_gram_apply_block`, fp64
  accumulation) -- sparse loadings touch only their support.  The centring
  is algebraic: (S - 1 mean') L = S L - 1 (mean' L); column means come from
  `gps_matvec_t` with 1/N weights.  Sequential deflation in
  explained_variance (pca.py:93-102) becomes, with Y = S V,
  s_j = Y_j - (mean' v_j) 1 - sum_{k<j} s_k (v_k' v_j).
* `knn_classify`: squared distances by the reference's expansion
  (|t|^2 - 2 t.s) + |s|^2 clamped at 0 and the first minimum per test row
  (`gps_knn_distances`); k > 1 selects the k nearest in (distance, index)
  order with a device selection kernel (`gps_knn_topk`), and the vote
  follows datasets.py:258-270 on the k selected labels.
* `pca_fit`: centring (`gps_matrix_center`) and the thin SVD by one-sided
  Jacobi on the device (`gps_matrix_svd`), sign-fixed by
  `deterministic_signs`; torch only moves buffers.
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import DataMatrix, as_data_matrix


@dataclass(frozen=True)
class PcaModel:
    """pca.py:16-22."""

    components: np.ndarray
    singular_values: np.ndarray
    mean: np.ndarray


def deterministic_signs(L):
    """Flip each column so its largest-magnitude entry is positive
    (pca.py:25-34)."""
    L = np.array(L, dtype=np.float64, copy=True)
    for j in range(L.shape[1]):
        i = int(np.argmax(np.abs(L[:, j])))
        if L[i, j] < 0:
            L[:, j] = -L[:, j]
    return L


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the recognition path needs a CUDA device (no CPU fallback)")
    return torch


def pca_fit(samples, m):
    """Top-m principal components of a samples x variables matrix
    (pca.py:37-54): the leading right singular vectors of the centred data,
    sign-fixed.  Centring (gps_matrix_center) and the thin SVD (one-sided
    Jacobi on the device, gps_matrix_svd) run in libgpspca_b200."""
    from .core import center_columns_with_means

    S = np.asarray(samples, dtype=np.float64)
    if S.ndim != 2:
        raise ValueError("samples must be a 2-d matrix")
    if not 1 <= m <= min(S.shape):
        raise ValueError(f"need 1 <= m <= min(#samples, #variables) = {min(S.shape)}")
    Ac, mean = center_columns_with_means(DataMatrix(S))
    r = min(S.shape)
    sigma = np.empty(r)
    V = np.empty((S.shape[1], r), order="F")
    sweeps = _native.C.c_int(0)
    _native.check(_native.lib().gps_matrix_svd(Ac.handle, _native.dptr(sigma), V.ctypes.data_as(_native._dp),
                                               _native.C.byref(sweeps)), "pca_fit SVD")
    return PcaModel(
        components=deterministic_signs(V[:, :m]),
        singular_values=sigma[:m].copy(),
        mean=mean,
    )


def _as_samples_matrix(samples):
    """Samples (N x F) as the engine's column-major p x n DataMatrix
    (p = N samples, n = F features): the same storage GP-SPCA fits on."""
    if isinstance(samples, DataMatrix):
        return samples
    S = np.asarray(samples)
    if S.ndim != 2:
        raise ValueError("samples must be a 2-d matrix")
    dtype = np.float32 if S.dtype == np.float32 else np.float64
    return as_data_matrix(S.astype(dtype, copy=False))


def _column_means(A):
    ones = np.full(A.p, 1.0 / A.p)
    out = np.empty(A.n)
    _native.check(_native.lib().gps_matvec_t(A.handle, _native.dptr(ones), _native.dptr(out)))
    return out


def _apply(A, L):
    # column-major n x m (= row-major m x n) in, column-major p x m out
    Lt = np.ascontiguousarray(np.asarray(L, dtype=np.float64).T)
    m = Lt.shape[0]
    Yt = np.empty((m, A.p))
    _native.check(_native.lib().gps_gram_apply_block(A.handle, _native.dptr(Lt), int(m), _native.dptr(Yt)))
    return Yt.T


def project(samples, loadings, mean=None):
    """Embed samples: (samples - mean) @ loadings (pca.py:57-71)."""
    A = _as_samples_matrix(samples)
    L = np.asarray(loadings, dtype=np.float64)
    squeeze = L.ndim == 1
    if squeeze:
        L = L[:, None]
    if A.n != L.shape[0]:
        raise ValueError(f"samples have {A.n} features but loadings expect {L.shape[0]}")
    mean = _column_means(A) if mean is None else np.asarray(mean, dtype=np.float64)
    Y = _apply(A, L) - (mean @ L)[None, :]
    return Y[:, 0] if squeeze else Y


def explained_variance(samples, loadings, zero_tol=1e-12):
    """Variance captured per component after sequential deflation of the
    earlier components (pca.py:74-103)."""
    A = _as_samples_matrix(samples)
    L = np.asarray(loadings, dtype=np.float64)
    if L.ndim == 1:
        L = L[:, None]
    if A.n != L.shape[0]:
        raise ValueError("samples and loadings disagree on the feature count")
    norms = np.linalg.norm(L, axis=0)
    nonzero = norms > zero_tol
    if np.any(np.abs(norms[nonzero] - 1.0) > 1e-9):
        raise ValueError("loading columns must be unit norm or zero")
    mean = _column_means(A)
    Y = _apply(A, L) - (mean @ L)[None, :]  # centred scores before deflation
    denom = max(A.p - 1, 1)
    out = np.zeros(L.shape[1])
    kept = []  # (scores s_k, loading v_k) of the nonzero components so far
    for j in range(L.shape[1]):
        if not nonzero[j]:
            continue
        v = L[:, j]
        s = Y[:, j].copy()
        for sk, vk in kept:
            s -= sk * float(vk @ v)
        out[j] = float(s @ s) / denom
        kept.append((s, v))
    return out


def knn_classify(train_embedding, train_labels, test_embedding, test_labels=None, k=1):
    """Nearest-neighbour prediction in the embedded space
    (datasets.py:223-275): Euclidean metric, distance ties to the lowest
    train index, majority vote for k > 1 with ties to the label of the
    nearest tied neighbour.  Returns (predictions, accuracy)."""
    train = np.asarray(train_embedding, dtype=np.float64)
    test = np.asarray(test_embedding, dtype=np.float64)
    train_labels = np.asarray(train_labels)
    if train.shape[0] == 0:
        raise ValueError("training set is empty")
    if train.ndim != 2 or test.ndim != 2 or train.shape[1] != test.shape[1]:
        raise ValueError("train and test embeddings must share the column count")
    if not 1 <= k <= train.shape[0]:
        raise ValueError("k must be between 1 and the training-set size")
    predictions = np.empty(test.shape[0], dtype=train_labels.dtype)
    if test.shape[0] == 0:
        accuracy = None if test_labels is None else float(np.mean(predictions == np.asarray(test_labels)))
        return predictions, accuracy
    torch = _torch()
    ctx = _native.context()
    dev = f"cuda:{ctx.device}"
    L = _native.lib()
    R, dim = train.shape
    trainT = torch.from_numpy(np.ascontiguousarray(train.T)).to(dev)
    ss = torch.empty(R, dtype=torch.float64, device=dev)
    train_rows = torch.from_numpy(np.ascontiguousarray(train)).to(dev)
    torch.cuda.synchronize(dev)
    _native.check(L.gps_row_sqnorms(ctx.handle, _native.C.c_void_p(train_rows.data_ptr()), R, dim,
                                    _native.C.c_void_p(ss.data_ptr())))
    step = max(1, min(int(2**22 // max(R, 1)), 65535 * 16))  # same chunking bound as the reference
    for lo in range(0, test.shape[0], step):
        chunk = torch.from_numpy(np.ascontiguousarray(test[lo:lo + step])).to(dev)
        T = chunk.shape[0]
        dist = torch.empty((T, R), dtype=torch.float64, device=dev)
        amin = torch.empty(T, dtype=torch.int64, device=dev)
        torch.cuda.synchronize(dev)
        _native.check(L.gps_knn_distances(
            ctx.handle, _native.C.c_void_p(chunk.data_ptr()), T, _native.C.c_void_p(trainT.data_ptr()), R, dim,
            _native.C.c_void_p(ss.data_ptr()), _native.C.c_void_p(dist.data_ptr()),
            _native.C.c_void_p(amin.data_ptr()) if k == 1 else None))
        if k == 1:
            predictions[lo:lo + T] = train_labels[amin.cpu().numpy()]
            continue
        idx = torch.empty((T, k), dtype=torch.int64, device=dev)
        _native.check(L.gps_knn_topk(ctx.handle, _native.C.c_void_p(dist.data_ptr()), T, R, k,
                                     _native.C.c_void_p(idx.data_ptr())))
        order = idx.cpu().numpy()
        for r in range(T):
            votes = train_labels[order[r]]
            labels, counts = np.unique(votes, return_counts=True)
            winners = labels[counts == counts.max()]
            if winners.size == 1:
                predictions[lo + r] = winners[0]
            else:
                for idx in order[r]:
                    if train_labels[idx] in winners:
                        predictions[lo + r] = train_labels[idx]
                        break
    accuracy = None
    if test_labels is not None:
        accuracy = float(np.mean(predictions == np.asarray(test_labels)))
    return predictions, accuracy

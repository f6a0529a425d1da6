"""The tensor-core block sweep only filters columns (margin delta_i, see
DESIGN.md "Why the margin is safe"); every column that can be active is
recomputed in fp64.  These instances put EVERY column within 1e-10 .. 1e-2
(relative) of a threshold, far inside the filter's own error, so any column
the filter wrongly dropped, or any approximate value that leaked into the
results, shows up as a support or weight difference against the fp64 oracle
on the same (storage-rounded) numbers."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")
from paper_1312_6182_b200.block import _block_sweep  # noqa: E402


def near_threshold_instance(p, n, m, gamma, mu, penalty, seed):
    """Columns a_i = X t_i + (I - X X') z_i with one component of t_i placed at
    its threshold times (1 +- 10^-k), k in [2, 10], and the others below it."""
    rng = np.random.default_rng(seed)
    Q, R = np.linalg.qr(rng.standard_normal((p, m)))
    X = Q * np.sign(np.diagonal(R))
    level = gamma / mu if penalty == "l1" else np.sqrt(gamma) / mu  # |c| at the threshold
    T = rng.uniform(-0.5, 0.5, (m, n)) * level[:, None]
    jstar = rng.integers(0, m, n)
    rel = np.power(10.0, -rng.uniform(2, 10, n)) * rng.choice([-1.0, 1.0], n)
    T[jstar, np.arange(n)] = level[jstar] * (1.0 + rel) * rng.choice([-1.0, 1.0], n)
    Z = rng.standard_normal((p, n))
    Z -= X @ (X.T @ Z)
    return X @ T + 3.0 * Z, X


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["fp32", "fp64"])
@pytest.mark.parametrize("penalty", ["l1", "l0"])
@pytest.mark.parametrize("m", [3, 10, 64])
@pytest.mark.parametrize("f64_path", ["tc", "cuda_core"])
def test_every_column_near_threshold(dtype, penalty, m, f64_path, monkeypatch):
    if dtype == np.float32 and f64_path == "cuda_core":
        pytest.skip("fp32 storage always takes the tensor-core filter")
    monkeypatch.setenv("GPSPCA_TC_F64_MIN_BYTES", "0" if f64_path == "tc" else "1e30")
    p, n = 512, 3000
    mu = np.linspace(1.0, 0.6, m)
    gamma = np.full(m, 2.0 if penalty == "l1" else 4.0)
    A, X = near_threshold_instance(p, n, m, gamma, mu, penalty, seed=m + (penalty == "l0"))
    A = A.astype(dtype)
    A64 = A.astype(np.float64)
    C = oracle.block_correlations(A64, X)
    W_ref = np.column_stack([oracle.threshold(mu[j] * C[:, j], gamma[j], penalty) for j in range(m)])
    f_ref = oracle.block_objective(C, gamma, mu, penalty)
    G_ref = oracle.block_gradient(A64, C, gamma, mu, penalty)
    f, G, W = _block_sweep(gps.DataMatrix(A, dtype=dtype), X, gamma, mu, penalty, want_w=True)
    assert (W_ref != 0).sum() > 0.2 * n  # the band is populated
    np.testing.assert_array_equal(W != 0, W_ref != 0)
    np.testing.assert_allclose(W, W_ref, rtol=1e-9, atol=1e-12 * np.abs(W_ref).max())
    assert f == pytest.approx(f_ref, rel=1e-10)
    np.testing.assert_allclose(G, G_ref, rtol=1e-9, atol=1e-11 * np.abs(G_ref).max())

"""Parity at BASELINE-like scale (SURVEY §8d "parity at scale"): full
single-unit solves on a quarter-size C2 instance and truncated block
trajectories on a C3-shaped slice, device vs the fp64 oracle on the same
(fp32-drawn) numbers."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")


def lowrank_plus_noise(p, n, factors, support, seed):
    """The C2/C3 distribution (reference datasets.py:278-309), fp32."""
    rng = np.random.default_rng(seed)
    means = rng.standard_normal((16, factors)) * 4.0
    latent = means[np.repeat(np.arange(16), p // 16)] + rng.standard_normal((p, factors))
    A = rng.standard_normal((p, n), dtype=np.float32)
    for f in range(factors):
        e = rng.standard_normal(support)
        e /= np.linalg.norm(e)
        A[:, f * support:(f + 1) * support] += np.outer(latent[:, f], e).astype(np.float32)
    return np.asfortranarray(A)


def near(c, gamma, penalty, rel):
    return (np.abs(np.abs(c) - gamma) <= rel * gamma) if penalty == "l1" else (np.abs(c * c - gamma) <= rel * gamma)


@pytest.fixture(scope="module")
def c2_quarter():
    A32 = lowrank_plus_noise(4096, 1 << 18, 5, 400, seed=7)
    return A32, gps.DataMatrix(A32)


@pytest.mark.parametrize("penalty", ["l0", "l1"])
def test_su_full_solve_quarter_c2(c2_quarter, penalty):
    A32, A = c2_quarter
    A64 = A32.astype(np.float64)
    g1 = 0.05 * float(A.norms.max())
    gamma = g1 if penalty == "l1" else g1 * g1
    loadings, report = gps.solve_single_unit(A, gps.SolverConfig(penalty=penalty, gamma=gamma, max_iter=60))
    z, hist, conv, x = oracle.su_solve(A64, gamma, penalty, max_iter=60)
    assert report.iterations == len(hist) - 1
    np.testing.assert_allclose(report.objective_history, hist, rtol=1e-9)
    zd = loadings.values[:, 0]
    diff = (zd != 0) != (z != 0)
    if diff.any():
        assert not (diff & ~near(A64.T @ x, gamma, penalty, 1e-6)).any()
    np.testing.assert_allclose(zd, z, rtol=1e-7, atol=1e-9)


@pytest.mark.parametrize("penalty", ["l1", "l0"])
def test_block_truncated_c3_slice(penalty):
    A32 = lowrank_plus_noise(4096, 1 << 16, 10, 400, seed=8)
    A = gps.DataMatrix(A32)
    A64 = A32.astype(np.float64)
    g1 = 0.05 * float(A.norms.max())
    gamma = g1 if penalty == "l1" else g1 * g1
    cfg = gps.SolverConfig(penalty=penalty, mode="block", m=10, gamma=gamma, max_iter=3)
    loadings, report = gps.solve_block(A, cfg)
    Z, hist, conv, X = oracle.block_solve(A64, 10, gamma, 1.0, penalty, max_iter=3)
    assert report.iterations == len(hist) - 1 == 3
    np.testing.assert_allclose(report.objective_history, hist, rtol=1e-9)
    C = A64.T @ X
    diff = (loadings.values != 0) != (Z != 0)
    # north star: identical supports except entries within 1e-6 gamma of the threshold (logged)
    assert not (diff & ~near(C, gamma, penalty, 1e-6)).any()
    if diff.any():
        print(f"near-threshold support differences: {int(diff.sum())}")
    np.testing.assert_allclose(loadings.values, Z, rtol=1e-7, atol=1e-9)

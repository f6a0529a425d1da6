"""Large-problem block paths: the tensor-core (tcgen05) candidate filter +
fp64 recomputation for fp32 storage, and the multi-CTA CholeskyQR2 polar step for
large p*m, each against the fp64 oracle and against the exact paths."""

import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stiefel(rng, p, m):
    Q, R = np.linalg.qr(rng.standard_normal((p, m)))
    return Q * np.sign(np.diagonal(R))


@pytest.mark.parametrize("p,n,m,pen", [(256, 1000, 16, "l1"), (512, 3000, 32, "l0"), (4096, 12000, 64, "l1"),
                                        (8192, 8192, 64, "l0"), (300, 777, 24, "l1"), (4128, 3001, 10, "l1"),
                                        (10000, 2000, 5, "l0"), (33, 500, 7, "l1"), (1000, 129, 40, "l0")])
@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["fp32", "fp64"])
def test_tensor_core_sweep_vs_oracle(p, n, m, pen, dtype, monkeypatch):
    monkeypatch.setenv("GPSPCA_TC_F64_MIN_BYTES", "0")  # fp64: the tensor-core path at every size
    rng = np.random.default_rng(p + m)
    A32 = rng.standard_normal((p, n)).astype(np.float32)
    A = gps.DataMatrix(A32.astype(dtype), dtype=dtype)
    X = _stiefel(rng, p, m)
    gamma = np.full(m, 2.0 if pen == "l1" else 4.0)
    mu = np.linspace(1.0, 0.6, m)
    A64 = A32.astype(np.float64)
    C = A64.T @ X
    f_ref = oracle.block_objective(C, gamma, mu, pen)
    G_ref = oracle.block_gradient(A64, C, gamma, mu, pen)
    f = (gps.objective_bl1 if pen == "l1" else gps.objective_bl0)(A, X, gamma, mu)
    G = gps.ascent_direction_block(A, X, gamma, mu, pen)
    assert f == pytest.approx(f_ref, rel=1e-11)
    assert np.abs(G - G_ref).max() <= 1e-11 * np.abs(G_ref).max()


@pytest.mark.parametrize("p,n,m,pen", [(4096, 12000, 64, "l1"), (300, 777, 24, "l0")])
def test_two_term_filter_vs_oracle(p, n, m, pen, monkeypatch):
    """The two-term X filter (GPSPCA_TC_XTERMS=2: x 2^14 = X1 + 2^-11 X2,
    narrower margin) gives the same exact results as the default one-term
    filter."""
    monkeypatch.setenv("GPSPCA_TC_XTERMS", "2")
    rng = np.random.default_rng(p + m + 1)
    A32 = rng.standard_normal((p, n)).astype(np.float32)
    A = gps.DataMatrix(A32)
    X = _stiefel(rng, p, m)
    gamma = np.full(m, 2.0 if pen == "l1" else 4.0)
    mu = np.linspace(1.0, 0.6, m)
    A64 = A32.astype(np.float64)
    C = A64.T @ X
    f_ref = oracle.block_objective(C, gamma, mu, pen)
    G_ref = oracle.block_gradient(A64, C, gamma, mu, pen)
    f = (gps.objective_bl1 if pen == "l1" else gps.objective_bl0)(A, X, gamma, mu)
    G = gps.ascent_direction_block(A, X, gamma, mu, pen)
    assert f == pytest.approx(f_ref, rel=1e-11)
    assert np.abs(G - G_ref).max() <= 1e-11 * np.abs(G_ref).max()


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["fp32", "fp64"])
def test_tensor_core_solve_vs_oracle(dtype, monkeypatch):
    monkeypatch.setenv("GPSPCA_TC_F64_MIN_BYTES", "0")
    rng = np.random.default_rng(5)
    A32 = rng.standard_normal((400, 5000)).astype(np.float32)
    A64 = A32.astype(np.float64)
    gamma = 0.1 * float(np.linalg.norm(A64, axis=0).max())
    cfg = gps.SolverConfig(penalty="l1", mode="block", m=16, gamma=gamma, max_iter=40)
    loadings, report = gps.solve_block(gps.DataMatrix(A32.astype(dtype), dtype=dtype), cfg)
    Z, hist, conv, X = oracle.block_solve(A64, 16, gamma, 1.0, "l1", max_iter=40)
    assert report.iterations == len(hist) - 1
    np.testing.assert_allclose(report.objective_history, hist, rtol=1e-9)
    assert np.array_equal(loadings.values != 0, Z != 0)
    np.testing.assert_allclose(loadings.values, Z, rtol=1e-7, atol=1e-9)


def _run_env(code, **env):
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                         env={**os.environ, **env}, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout


POLAR_CODE = r"""
import numpy as np, json, sys
sys.path.insert(0, '.')
import paper_1312_6182_b200 as gps
rng = np.random.default_rng(11)
A = rng.standard_normal((4096, 6000))
g = 0.05 * float(np.linalg.norm(A, axis=0).max())
_, r = gps.solve_block(gps.DataMatrix(A), gps.SolverConfig(penalty='l1', mode='block', m=10, gamma=g, max_iter=25))
print(json.dumps(r.objective_history))
"""


def test_cholqr2_polar_matches_householder_polar():
    import json

    big = json.loads(_run_env(POLAR_CODE).strip().splitlines()[-1])
    hh = json.loads(_run_env(POLAR_CODE, GPSPCA_HH_POLAR="1").strip().splitlines()[-1])
    assert len(big) == len(hh)
    np.testing.assert_allclose(big, hh, rtol=1e-10)


def test_rank_collapse_through_large_paths():
    # rank-5 data, m = 16 components, gamma = 0: G has rank 5 at the first step;
    # the CholeskyQR2 polar must hand over to the exact path and report it.
    rng = np.random.default_rng(12)
    A32 = (rng.standard_normal((4096, 5)) @ rng.standard_normal((5, 3000))).astype(np.float32)
    cfg = gps.SolverConfig(penalty="l1", mode="block", m=16, gamma=0.0, init="random_orthonormal", seed=0)
    with pytest.raises(gps.RankDeficiencyError) as err:
        gps.solve_block(gps.DataMatrix(A32), cfg)
    assert err.value.rank == 5 and err.value.iteration == 0

"""Round-2 parity fixtures on the GPU (tests/golden/solves_hard.json and
polar.json, produced by running the reference: make_golden.py --hard).

- Block solves at m = 32 / 64 on a 256 x 4096 rank-64 matrix: the C4 code
  paths (tensor-core refine / update with 64 padded components, the
  CholeskyQR2 + Newton-Schulz polar step with its Stiefel check, CholeskyQR2
  initialisation at p m >= 4096), dense activity (random starts with small
  gamma keep ~2000 of 4096 columns active), rank loss inside the loop, in
  both storage dtypes, against the reference at 1e-12 with identical
  iteration counts and supports.  Every iterate's ||X'X - I||_F is recorded
  and must meet the reference's 1e-10 (block.py:149, core.py:113-129).
- Near-collinear / duplicated max-norm columns at init: the reference's
  Householder rule (block.py:162-168) decides, not a Cholesky breakdown.
- solve_multi_sequential with refine=True (refine on the deflated matrix).
- polar_projection on G = U diag(s) V' with kappa = 10 .. 1e7 and the
  rank-cutoff cases, through the exact one-CTA path AND the loop's
  CholeskyQR2 path (which must hand ill-conditioned G to the exact path).
"""

import base64
import json
import os

import numpy as np
import pytest

from golden_cases import case_matrix, dense_z

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(HERE, "solves_hard.json")) as fh:
    HARD = json.load(fh)["cases"]
with open(os.path.join(HERE, "polar.json")) as fh:
    POLAR = json.load(fh)["cases"]

BLOCK = [c for c in HARD if c["solver"] == "block"]
MULTI = [c for c in HARD if c["solver"] == "multi_sequential"]


def unb64(d):
    return np.frombuffer(base64.b64decode(d["data"]), dtype=np.float64).reshape(d["shape"], order="F")


def _cfg(case):
    return gps.SolverConfig(penalty=case["penalty"], mode="block", m=case["m"], gamma=case["gamma"],
                            mu=case["mu"], **case["config"])


def _check_support(loadings, Zg, report):
    """Supports identical except the logged near-threshold entries."""
    mine, ref = loadings.values != 0, Zg != 0
    diff = np.argwhere(mine != ref)
    for i, j in diff:
        assert i in set(report.near_threshold[j].tolist()), (int(i), int(j))


def _hist_rtol(case):
    # near-collinear starts: a backward-stable QR determines the second
    # column of Q of a kappa ~ 1 / rel matrix only up to ~kappa eps, so X_0
    # -- and f_0 -- differ from the reference's LAPACK QR at that level
    # (measured: 1.5e-9 relative in f_0 at rel = 1e-12); bound 1e-8
    nearcol = case["recipe"]["kind"] == "nearcol" and case["recipe"]["rel"] > 0
    return 1e-8 if nearcol else 1e-12


def _store(case):
    # the near-collinear recipes are built in fp64 and only exist in fp64
    return [np.float64] if case["recipe"]["kind"] == "nearcol" else [np.float64, np.float32]


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["fp64", "fp32"])
@pytest.mark.parametrize("case", BLOCK, ids=[c["name"] for c in BLOCK])
def test_hard_block_solves(case, dtype):
    if dtype not in _store(case):
        pytest.skip("fp64-only recipe")
    A = gps.DataMatrix(case_matrix(case).astype(dtype))
    cfg = _cfg(case)
    if "init_error" in case:
        with pytest.raises(ValueError, match="rank deficient"):
            gps.solve_block(A, cfg)
        return
    if "rank_error" in case:
        with pytest.raises(gps.RankDeficiencyError) as err:
            gps.solve_block(A, cfg)
        assert err.value.rank == case["rank_error"]["rank"]
        assert err.value.iteration == case["rank_error"]["iteration"]
        np.testing.assert_allclose(err.value.history, case["rank_error"]["history"], rtol=_hist_rtol(case))
        return
    loadings, report = gps.solve_block(A, cfg)
    assert report.iterations == case["iterations"]
    assert report.converged == case["converged"]
    np.testing.assert_allclose(report.objective_history, case["history"], rtol=1e-12, atol=1e-13)
    Zg = dense_z(case, A.n)
    _check_support(loadings, Zg, report)
    np.testing.assert_allclose(loadings.values, Zg, rtol=1e-10, atol=1e-12)
    st = report.stiefel_errors
    assert len(st) == report.iterations + 1
    assert max(st) <= 1e-10, max(st)


@pytest.mark.parametrize("case", MULTI, ids=[c["name"] for c in MULTI])
def test_hard_multi_refine(case):
    A = gps.DataMatrix(case_matrix(case).astype(np.float32))
    cfg = gps.SolverConfig(penalty=case["penalty"], gamma=case["gamma"], m=case["m"], **case["config"])
    loadings, report = gps.solve_multi_sequential(A, cfg)
    assert report.iterations == case["iterations"]
    for mine, ref in zip(report.component_histories, case["histories"]):
        np.testing.assert_allclose(mine, ref, rtol=1e-10, atol=1e-12)
    Zg = dense_z(case, A.n)
    _check_support(loadings, Zg, report)
    np.testing.assert_allclose(loadings.values, Zg, rtol=1e-9, atol=1e-11)


def _polar_tol(case):
    # the polar factor moves by ~ eps * kappa under rounding-level changes of G
    s = np.asarray(case["s"])
    kappa = s[0] / s[-1] if s[-1] > 0 else np.inf
    return max(1e-12, 100 * kappa * np.finfo(np.float64).eps)


@pytest.mark.parametrize("case", POLAR, ids=[c["name"] for c in POLAR])
def test_polar_exact_path(case):
    G = unb64(case["G"])
    if "rank_error" in case:
        with pytest.raises(gps.RankDeficiencyError) as err:
            gps.polar_projection(G)
        assert err.value.rank == case["rank_error"]["rank"]
        return
    X = gps.polar_projection(G).values
    Xr = unb64(case["X"])
    assert np.max(np.abs(X - Xr)) <= _polar_tol(case)
    assert np.linalg.norm(X.T @ X - np.eye(X.shape[1])) <= 1e-10


@pytest.mark.parametrize("case", POLAR, ids=[c["name"] for c in POLAR])
def test_polar_cholqr2_path(case):
    """The in-loop multi-CTA step: CholeskyQR2 only where its result is a
    valid StiefelPoint (kappa_F(R1) <= 1e5, R2 ~ I, Gram check), the exact
    path everywhere else -- same rank decisions, same X within tolerance."""
    from paper_1312_6182_b200.block import _polar_cholqr2

    G = unb64(case["G"])
    if "rank_error" in case:
        with pytest.raises(gps.RankDeficiencyError) as err:
            _polar_cholqr2(G)
        assert err.value.rank == case["rank_error"]["rank"]
        return
    X, st, exact = _polar_cholqr2(G)
    Xr = unb64(case["X"])
    kappa = case["s"][0] / case["s"][-1]
    if kappa >= 1e7:
        assert exact, "kappa = 1e7 must take the exact path"
    if kappa <= 1e3:
        assert not exact, "well-conditioned G keeps the CholeskyQR2 path"
    assert st <= 1e-10
    assert np.max(np.abs(X - Xr)) <= _polar_tol(case)


def test_polar_cholqr2_matches_exact_on_the_loop_shapes():
    """C3 / C4 polar shapes (4096 x 10, 8192 x 64) at moderate kappa: the fast
    path agrees with the exact path to 1e-12."""
    from paper_1312_6182_b200.block import _polar_cholqr2

    rng = np.random.default_rng(3)
    for p, m in ((4096, 10), (8192, 64)):
        G = rng.standard_normal((p, m)) @ np.diag(np.logspace(0, -2, m))
        X, st, exact = _polar_cholqr2(G)
        assert not exact and st <= 1e-13
        Xe = gps.polar_projection(G).values
        assert np.max(np.abs(X - Xe)) <= 1e-12

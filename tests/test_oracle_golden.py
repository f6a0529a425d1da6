"""Pin the CPU oracle (oracle/gpower.py) to the reference's own outputs.

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py); here the restatement must reproduce them:
identical iteration counts and supports, histories and loadings to 1e-10.
"""

import numpy as np
import pytest

import oracle
from golden_cases import case_matrix, dense_z, load_kernels, load_solves

CASES = load_solves()


def _cfg(case):
    return dict(case.get("config", {}))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference(case):
    A = case_matrix(case)
    n = A.shape[1]
    cfg = _cfg(case)
    if case["solver"] == "single_unit":
        z, hist, conv, x = oracle.su_solve(A, case["gamma"], case["penalty"], **cfg)
        assert len(hist) - 1 == case["iterations"]
        assert conv == case["converged"]
        np.testing.assert_allclose(hist, case["history"], rtol=1e-10, atol=1e-12)
        Zg = dense_z(case, n)
        assert np.array_equal(np.nonzero(z)[0], np.nonzero(Zg[:, 0])[0])
        np.testing.assert_allclose(z, Zg[:, 0], rtol=1e-9, atol=1e-10)
    elif case["solver"] == "multi_sequential":
        gammas = [case["gamma"]] * case["m"]
        Z, hists, conv = oracle.multi_sequential(A, gammas, case["penalty"], **cfg)
        assert sum(len(h) - 1 for h in hists) == case["iterations"]
        for h, hg in zip(hists, case["histories"]):
            np.testing.assert_allclose(h, hg, rtol=1e-10, atol=1e-12)
        Zg = dense_z(case, n)
        assert np.array_equal(Z != 0, Zg != 0)
        np.testing.assert_allclose(Z, Zg, rtol=1e-9, atol=1e-10)
    else:
        kw = dict(cfg)
        init = kw.pop("init", "max_norm_column")
        if "rank_error" in case:
            with pytest.raises(oracle.OracleRankDeficiency) as err:
                oracle.block_solve(A, case["m"], case["gamma"], case["mu"], case["penalty"],
                                   init=init, **kw)
            assert err.value.rank == case["rank_error"]["rank"]
            assert err.value.iteration == case["rank_error"]["iteration"]
            return
        Z, hist, conv, X = oracle.block_solve(A, case["m"], case["gamma"], case["mu"],
                                              case["penalty"], init=init, **kw)
        assert len(hist) - 1 == case["iterations"]
        np.testing.assert_allclose(hist, case["history"], rtol=1e-10, atol=1e-12)
        Zg = dense_z(case, n)
        assert np.array_equal(Z != 0, Zg != 0)
        np.testing.assert_allclose(Z, Zg, rtol=1e-8, atol=1e-9)


def test_oracle_kernel_vectors():
    k = load_kernels()
    A = case_matrix(k)
    x = np.array(k["x"])
    c = A.T @ x
    np.testing.assert_allclose(c, k["matvec_t"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(A @ np.array(k["coef"]), k["gram_apply"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.column_norms(A), k["column_norms"], rtol=1e-14)
    for pen, gam in (("l1", 0.5), ("l0", 0.25)):
        np.testing.assert_allclose(oracle.su_gradient(A, c, gam, pen) / 2.0,
                                   k[f"threshold_accumulate_{pen}"], rtol=1e-12, atol=1e-12)
        assert oracle.su_objective(c, gam, pen) == pytest.approx(k[f"objective_{pen}"], rel=1e-13)
        np.testing.assert_allclose(oracle.su_recover(A, x, gam, pen), k[f"recover_{pen}"],
                                   rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(oracle.polar(np.array(k["polar_G"])), k["polar_X"], atol=1e-13)
    X = np.array(k["block_X"])
    C = oracle.block_correlations(A, X)
    for pen in ("l1", "l0"):
        assert oracle.block_objective(C, k["block_gamma"], k["block_mu"], pen) == pytest.approx(
            k[f"objective_bl{pen[1]}"], rel=1e-13)
        np.testing.assert_allclose(oracle.block_gradient(A, C, k["block_gamma"], k["block_mu"], pen),
                                   k[f"ascent_block_{pen}"], rtol=1e-12, atol=1e-12)


def test_threshold_tie_is_inactive():
    # parallel.py:127 / reference test_parallel.py:109-114
    assert oracle.threshold(np.array([1.0, 0.0]), 1.0, "l0").tolist() == [0.0, 0.0]


def test_chunked_oracle_matches_whole_matrix_oracle():
    """oracle/chunked.py (the full-size checker) agrees with the pinned
    whole-matrix restatement on the C1 golden instance, both loops."""
    from oracle.chunked import ChunkedA, block_solve_chunked, max_norm_start, su_iterate_chunked

    case = next(c for c in load_solves() if c["name"] == "c1_bl1_m10")
    A = case_matrix(case)
    H = ChunkedA(np.asfortranarray(A.astype(np.float32)), chunk=97, workers=4)
    np.testing.assert_allclose(H.norms(), oracle.column_norms(A), rtol=1e-14)
    X0, _ = max_norm_start(H, 10)
    np.testing.assert_allclose(X0, oracle.block_initial_point(A, 10), atol=1e-12)
    C, hist, conv, X = block_solve_chunked(H, 10, case["gamma"], 1.0, "l1", 1e-6, 1000, X0)
    assert len(hist) - 1 == case["iterations"]
    np.testing.assert_allclose(hist, case["history"], rtol=1e-11)
    su = next(c for c in load_solves() if c["name"] == "c1_sl1")
    norms = H.norms()
    i = int(np.argmax(norms))
    x, h, conv, c = su_iterate_chunked(H, H.column(i) / norms[i], su["gamma"], "l1", 1e-6, 1000)
    assert len(h) - 1 == su["iterations"]
    np.testing.assert_allclose(h, su["history"], rtol=1e-11)

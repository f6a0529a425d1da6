"""GPU parity suite for the block path (calls through libgpspca_b200).

Both storage modes compute in fp64 (fp32 storage: the tensor-core sweep only
filters columns, every column that can be active is recomputed in fp64) and
must match the reference's golden outputs to 1e-12 (histories and loadings)
with identical iteration counts and supports; measured worst case 8.2e-15
(profiles/parity_margins_r1.txt).
"""

import numpy as np
import pytest

import oracle
from golden_cases import case_matrix, dense_z, load_kernels, load_solves

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")

BLOCK_CASES = [c for c in load_solves() if c["solver"] == "block"]


def _cfg(case):
    kw = dict(case["config"])
    return gps.SolverConfig(penalty=case["penalty"], mode="block", m=case["m"], gamma=case["gamma"],
                            mu=case["mu"], **kw)


def random_stiefel(rng, p, m):
    Q, R = np.linalg.qr(rng.standard_normal((p, m)))
    return Q * np.sign(np.diagonal(R))


@pytest.mark.parametrize("f64_path", ["cuda_core", "tc"])
@pytest.mark.parametrize("case", BLOCK_CASES, ids=[c["name"] for c in BLOCK_CASES])
def test_solve_block_golden_fp64(case, f64_path, monkeypatch):
    # small fp64 problems take the CUDA-core sweep by default; force each path
    monkeypatch.setenv("GPSPCA_TC_F64_MIN_BYTES", "1e30" if f64_path == "cuda_core" else "0")
    A = gps.DataMatrix(case_matrix(case), dtype=np.float64)
    cfg = _cfg(case)
    if "rank_error" in case:
        with pytest.raises(gps.RankDeficiencyError) as err:
            gps.solve_block(A, cfg)
        assert err.value.rank == case["rank_error"]["rank"]
        assert err.value.iteration == case["rank_error"]["iteration"]
        np.testing.assert_allclose(err.value.history, case["rank_error"]["history"], rtol=1e-12)
        return
    loadings, report = gps.solve_block(A, cfg)
    assert report.iterations == case["iterations"]
    assert report.converged == case["converged"]
    np.testing.assert_allclose(report.objective_history, case["history"], rtol=1e-12, atol=1e-13)
    Zg = dense_z(case, A.n)
    assert np.array_equal(loadings.values != 0, Zg != 0)
    np.testing.assert_allclose(loadings.values, Zg, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("case", [c for c in BLOCK_CASES if "rank_error" not in c],
                         ids=[c["name"] for c in BLOCK_CASES if "rank_error" not in c])
def test_solve_block_golden_fp32(case):
    # fp32 storage: the tensor-core sweep only filters columns; every column
    # that can be active is recomputed in fp64 (T1x), so the fp32 path is held
    # to the fp64 bar: same iterations, supports, histories and loadings.
    A64 = case_matrix(case)
    A = gps.DataMatrix(A64.astype(np.float32))
    loadings, report = gps.solve_block(A, _cfg(case))
    assert report.iterations == case["iterations"]
    assert report.converged == case["converged"]
    np.testing.assert_allclose(report.objective_history, case["history"], rtol=1e-12, atol=1e-13)
    Zg = dense_z(case, A.n)
    assert np.array_equal(loadings.values != 0, Zg != 0)
    np.testing.assert_allclose(loadings.values, Zg, rtol=1e-12, atol=1e-13)


def test_solve_block_golden_fp32_rank_error():
    case = next(c for c in BLOCK_CASES if "rank_error" in c)
    A = gps.DataMatrix(case_matrix(case).astype(np.float32))
    with pytest.raises(gps.RankDeficiencyError) as err:
        gps.solve_block(A, _cfg(case))
    assert err.value.rank == case["rank_error"]["rank"]
    assert err.value.iteration == case["rank_error"]["iteration"]
    np.testing.assert_allclose(err.value.history, case["rank_error"]["history"], rtol=1e-12)


class TestBlockKernels:
    k = load_kernels()

    @pytest.fixture(params=[np.float64, np.float32], ids=["fp64", "fp32"])
    def A(self, request):
        return gps.DataMatrix(case_matrix(self.k).astype(request.param), dtype=request.param)

    def test_objectives(self, A):
        tol = 1e-12
        X = np.array(self.k["block_X"])
        for pen, fn in (("l1", gps.objective_bl1), ("l0", gps.objective_bl0)):
            assert fn(A, X, self.k["block_gamma"], self.k["block_mu"]) == pytest.approx(
                self.k[f"objective_bl{pen[1]}"], rel=tol)

    def test_ascent(self, A):
        rtol, atol = 1e-12, 1e-12
        X = np.array(self.k["block_X"])
        for pen in ("l1", "l0"):
            np.testing.assert_allclose(
                gps.ascent_direction_block(A, X, self.k["block_gamma"], self.k["block_mu"], pen),
                self.k[f"ascent_block_{pen}"], rtol=rtol, atol=atol)

    def test_polar(self):
        X = gps.polar_projection(np.array(self.k["polar_G"])).values
        np.testing.assert_allclose(X, self.k["polar_X"], atol=1e-12)


class TestReferenceBehaviour:
    """Known answers / invariants of the reference suite (test_block.py)."""

    def test_orthonormal_input_is_fixed(self):
        Q = random_stiefel(np.random.default_rng(34), 5, 3)
        assert np.allclose(gps.polar_projection(Q).values, Q, atol=1e-12)

    def test_positive_diagonal(self):
        G = np.zeros((4, 2))
        G[0, 0], G[1, 1] = 3.0, 2.0
        assert np.allclose(gps.polar_projection(G).values, np.eye(4)[:, :2], atol=1e-12)

    def test_feasible_to_tight_tolerance(self):
        rng = np.random.default_rng(36)
        for _ in range(50):
            X = gps.polar_projection(rng.standard_normal((7, 3))).values
            assert np.linalg.norm(X.T @ X - np.eye(3)) <= 1e-10

    def test_rank_deficient_raises_with_rank(self):
        G = np.zeros((4, 2))
        G[:, 0] = [1.0, 2.0, 3.0, 4.0]
        with pytest.raises(gps.RankDeficiencyError) as err:
            gps.polar_projection(G)
        assert err.value.rank == 1 and err.value.required == 2

    def test_m_one_equals_single_unit_exactly(self):
        rng = np.random.default_rng(32)
        A = rng.standard_normal((4, 7))
        x = rng.standard_normal(4)
        x /= np.linalg.norm(x)
        for penalty, single in (("l1", gps.ascent_direction_sl1), ("l0", gps.ascent_direction_sl0)):
            G = gps.ascent_direction_block(A, x, (0.2,), (1.0,), penalty)
            assert np.array_equal(G[:, 0], single(A, x, 0.2))

    def test_identity_example(self):
        G = gps.ascent_direction_block(np.eye(2), np.eye(2), (0.0, 0.0), (1.0, 1.0), "l1")
        assert np.allclose(G, 2.0 * np.eye(2))

    def test_m_one_matches_single_unit(self):
        rng = np.random.default_rng(37)
        A = rng.standard_normal((5, 8))
        for penalty in ("l1", "l0"):
            zb, rb = gps.solve_block(A, gps.SolverConfig(penalty=penalty, mode="block", m=1, gamma=0.2, tol=1e-12))
            zs, rs = gps.solve_single_unit(A, gps.SolverConfig(penalty=penalty, m=1, gamma=0.2, tol=1e-12))
            assert abs(rb.objective_history[-1] - rs.objective_history[-1]) <= 1e-8
            diff = min(np.abs(zb.values[:, 0] - zs.values[:, 0]).max(),
                       np.abs(zb.values[:, 0] + zs.values[:, 0]).max())
            assert diff <= 1e-6

    def test_symmetric_instance_objective_three(self):
        cfg = gps.SolverConfig(penalty="l1", mode="block", m=3, gamma=0.0, init="random_orthonormal", seed=0,
                               tol=1e-12)
        _, report = gps.solve_block(np.eye(3), cfg)
        assert report.objective_history[-1] == pytest.approx(3.0, abs=1e-8)

    def test_gamma_zero_distinct_mu_aligns_axes(self):
        A = np.diag([3.0, 2.0, 1.0])
        cfg = gps.SolverConfig(penalty="l1", mode="block", m=2, gamma=0.0, mu=(1.0, 0.5),
                               init="random_orthonormal", seed=3, tol=1e-14, max_iter=20000)
        loadings, _ = gps.solve_block(A, cfg)
        assert abs(loadings.values[0, 0]) >= 1 - 1e-6
        assert abs(loadings.values[1, 1]) >= 1 - 1e-6

    @pytest.mark.parametrize("penalty", ["l1", "l0"])
    def test_monotone_history(self, penalty):
        rng = np.random.default_rng(38)
        for _ in range(20):
            p = int(rng.integers(3, 8))
            A = rng.standard_normal((p, int(rng.integers(3, 12))))
            cfg = gps.SolverConfig(penalty=penalty, mode="block", m=2, gamma=float(rng.uniform(0, 0.3)),
                                   init="random_orthonormal", seed=int(rng.integers(1 << 16)))
            try:
                _, report = gps.solve_block(A, cfg)
                history = report.objective_history
            except gps.RankDeficiencyError as err:
                history = err.history
            assert np.all(np.diff(history) >= -1e-12)

    def test_permutation_equivariance(self):
        rng = np.random.default_rng(39)
        A = rng.standard_normal((5, 9))
        X0 = random_stiefel(rng, 5, 3)
        gamma, mu, perm = (0.05, 0.1, 0.2), (1.0, 0.8, 0.6), [2, 0, 1]
        Z, _ = gps.solve_block(A, gps.SolverConfig(penalty="l1", mode="block", m=3, gamma=gamma, mu=mu,
                                                   init="user_supplied", x0=X0, tol=1e-12, max_iter=5000))
        Zp, _ = gps.solve_block(A, gps.SolverConfig(penalty="l1", mode="block", m=3,
                                                    gamma=tuple(gamma[i] for i in perm),
                                                    mu=tuple(mu[i] for i in perm), init="user_supplied",
                                                    x0=X0[:, perm], tol=1e-12, max_iter=5000))
        np.testing.assert_allclose(Zp.values, Z.values[:, perm], atol=1e-10)

    def test_rejects_bad_m_and_mode(self):
        with pytest.raises(ValueError):
            gps.solve_block(np.eye(3), gps.SolverConfig(mode="block", m=4))
        with pytest.raises(ValueError):
            gps.solve_block(np.eye(3), gps.SolverConfig(mode="single_unit"))

    def test_stiefel_feasibility_every_polar(self):
        # acceptance criterion 5 analogue: polar outputs stay on the manifold
        rng = np.random.default_rng(105)
        worst = 0.0
        for _ in range(30):
            G = rng.standard_normal((int(rng.integers(3, 20)), 3))
            X = gps.polar_projection(G).values
            worst = max(worst, np.linalg.norm(X.T @ X - np.eye(3)))
        assert worst <= 1e-10


class TestLargeBlock:
    def test_block_sweep_c3_like_vs_oracle(self):
        rng = np.random.default_rng(9)
        p, n, m = 4096, 1 << 14, 10
        A32 = rng.standard_normal((p, n), dtype=np.float32)
        A = gps.DataMatrix(np.asfortranarray(A32))
        X = random_stiefel(rng, p, m)
        gamma = np.full(m, 2.5)  # |c| ~ N(0, 1): a few percent of the columns activate
        mu = np.linspace(1.0, 0.5, m)
        A64 = A32.astype(np.float64)
        C = oracle.block_correlations(A64, X)
        for pen in ("l1", "l0"):
            g = gamma if pen == "l1" else gamma ** 2
            f_ref = oracle.block_objective(C, g, mu, pen)
            G_ref = oracle.block_gradient(A64, C, g, mu, pen)
            G = gps.ascent_direction_block(A, X, g, mu, pen)
            f = (gps.objective_bl1 if pen == "l1" else gps.objective_bl0)(A, X, g, mu)
            # fp32 storage: tensor-core filter + fp64 recomputation of the candidates
            assert f_ref > 0 and f == pytest.approx(f_ref, rel=1e-11)
            np.testing.assert_allclose(G, G_ref, rtol=1e-10, atol=1e-11 * np.abs(G_ref).max())

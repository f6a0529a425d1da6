"""GPU parity suite for the single-unit path (calls through libgpspca_b200).

Oracle: the reference's own outputs (tests/golden/*.json, produced by
running /root/reference) and the NumPy restatement in oracle/.  Inputs are
float32 draws widened to float64 for the reference, so both storage modes
of the device (fp32 storage / fp64 storage, fp64 arithmetic either way)
see exactly the reference's numbers.  Tolerances: supports identical
except entries within 1e-6*gamma of the threshold (reported),
histories and loadings to 1e-12 -- tighter than the 1e-4 fp32 / 1e-10 fp64
bar because the device computes in fp64 in both modes (measured worst case
8.2e-15, profiles/parity_margins_r1.txt).
"""

import numpy as np
import pytest

import oracle
from golden_cases import case_matrix, dense_z, load_kernels, load_solves

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")

SU_CASES = [c for c in load_solves() if c["solver"] == "single_unit"]
MULTI_CASES = [c for c in load_solves() if c["solver"] == "multi_sequential"]


def _store(A, dtype):
    return gps.DataMatrix(A.astype(dtype), dtype=dtype)


def near_threshold(c, gamma, penalty, rel=1e-6):
    """Columns whose activation is decided within rel*gamma of the threshold."""
    if penalty == "l1":
        return np.abs(np.abs(c) - gamma) <= rel * max(gamma, 1e-300)
    return np.abs(c * c - gamma) <= rel * max(gamma, 1e-300)


def assert_support_equal(z_dev, z_ref, c_ref, gamma, penalty):
    diff = (z_dev != 0) != (z_ref != 0)
    if diff.any():
        allowed = near_threshold(c_ref, gamma, penalty)
        bad = diff & ~allowed
        assert not bad.any(), f"support differs at {np.flatnonzero(bad)[:10]}"


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["fp64", "fp32"])
@pytest.mark.parametrize("case", SU_CASES, ids=[c["name"] for c in SU_CASES])
def test_solve_single_unit_golden(case, dtype):
    A = case_matrix(case)
    cfg = gps.SolverConfig(penalty=case["penalty"], gamma=case["gamma"], **case["config"])
    loadings, report = gps.solve_single_unit(_store(A, dtype), cfg)
    assert report.iterations == case["iterations"]
    assert report.converged == case["converged"]
    np.testing.assert_allclose(report.objective_history, case["history"], rtol=1e-12, atol=1e-13)
    zg = dense_z(case, A.shape[1])[:, 0]
    z = loadings.values[:, 0]
    c_ref = A.T @ np.array(case["x"]) if case["x"] is not None else np.zeros(A.shape[1])
    assert_support_equal(z, zg, c_ref, case["gamma"], case["penalty"])
    np.testing.assert_allclose(z, zg, rtol=1e-12, atol=1e-13)
    assert report.kernel_launches > 0 or case["iterations"] == 0


@pytest.mark.parametrize("case", MULTI_CASES, ids=[c["name"] for c in MULTI_CASES])
def test_solve_multi_sequential_golden(case):
    A = case_matrix(case)
    cfg = gps.SolverConfig(penalty=case["penalty"], gamma=case["gamma"], m=case["m"], **case["config"])
    loadings, report = gps.solve_multi_sequential(_store(A, np.float32), cfg)
    assert report.iterations == case["iterations"]
    for h, hg in zip(report.component_histories, case["histories"]):
        np.testing.assert_allclose(h, hg, rtol=1e-12, atol=1e-13)
    Zg = dense_z(case, A.shape[1])
    assert np.array_equal(loadings.values != 0, Zg != 0)
    np.testing.assert_allclose(loadings.values, Zg, rtol=1e-12, atol=1e-13)


class TestKernelSeam:
    """parallel.py:85-142 known answers (tests/golden/kernels.json)."""

    k = load_kernels()

    @pytest.fixture(params=[np.float64, np.float32], ids=["fp64", "fp32"])
    def A(self, request):
        return _store(case_matrix(self.k), request.param)

    def test_matvec_t(self, A):
        np.testing.assert_allclose(gps.par_matvec_t(A, self.k["x"]), self.k["matvec_t"], rtol=1e-12, atol=1e-13)

    def test_gram_apply(self, A):
        np.testing.assert_allclose(gps.par_gram_apply(A, self.k["coef"]), self.k["gram_apply"],
                                   rtol=1e-12, atol=1e-12)

    @pytest.mark.parametrize("pen,gam", [("l1", 0.5), ("l0", 0.25)])
    def test_threshold_accumulate(self, A, pen, gam):
        c = np.array(self.k["matvec_t"])
        np.testing.assert_allclose(gps.par_threshold_accumulate(A, c, gam, pen),
                                   self.k[f"threshold_accumulate_{pen}"], rtol=1e-12, atol=1e-12)

    @pytest.mark.parametrize("pen,gam", [("l1", 0.5), ("l0", 0.25)])
    def test_objective_ascent_recover(self, A, pen, gam):
        x = self.k["x"]
        obj = gps.objective_sl1 if pen == "l1" else gps.objective_sl0
        asc = gps.ascent_direction_sl1 if pen == "l1" else gps.ascent_direction_sl0
        rec = gps.recover_pattern_sl1 if pen == "l1" else gps.recover_pattern_sl0
        assert obj(A, x, gam) == pytest.approx(self.k[f"objective_{pen}"], rel=1e-12)
        np.testing.assert_allclose(asc(A, x, gam), self.k[f"ascent_{pen}"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(rec(A, x, gam), self.k[f"recover_{pen}"], rtol=1e-11, atol=1e-13)

    def test_column_norms(self, A):
        np.testing.assert_allclose(gps.column_norms(A), self.k["column_norms"], rtol=1e-14)


class TestReferenceBehaviour:
    """Known answers and invariants from the reference's own suite
    (test_single_unit.py / test_parallel.py), run on the device."""

    def test_identity_matvec(self):
        assert np.array_equal(gps.par_matvec_t(np.eye(3), np.array([1.0, 2.0, 3.0])), [1.0, 2.0, 3.0])

    def test_zero_vector(self):
        A = np.random.default_rng(0).standard_normal((5, 9))
        assert np.array_equal(gps.par_matvec_t(A, np.zeros(5)), np.zeros(9))

    def test_single_active_column(self):
        out = gps.par_threshold_accumulate(np.eye(2), np.array([1.0, 0.0]), 0.25, "l1")
        assert np.array_equal(out, [0.75, 0.0])

    def test_l0_tie_is_inactive(self):
        out = gps.par_threshold_accumulate(np.eye(2), np.array([1.0, 0.0]), 1.0, "l0")
        assert np.array_equal(out, np.zeros(2))

    def test_dimension_mismatch(self):
        with pytest.raises(ValueError):
            gps.par_matvec_t(np.eye(3), np.ones(4))

    def test_nonfinite_rejected(self):
        A = np.ones((4, 5))
        A[2, 3] = np.nan
        with pytest.raises(ValueError):
            gps.DataMatrix(A)
        A[2, 3] = np.inf
        with pytest.raises(ValueError):
            gps.DataMatrix(A.astype(np.float32))

    def test_sl1_hand_derived(self):
        z = gps.recover_pattern_sl1(np.array([[1.0, 0.6], [0.0, 0.8]]), np.array([1.0, 0.0]), 0.5)
        np.testing.assert_allclose(z, np.array([5.0, 1.0]) / np.sqrt(26.0), atol=1e-12)

    def test_gamma_zero_recovers_leading_singular_vector(self):
        rng = np.random.default_rng(16)
        for penalty in ("l1", "l0"):
            A = rng.standard_normal((6, 10))
            cfg = gps.SolverConfig(penalty=penalty, gamma=0.0, tol=1e-14, max_iter=5000)
            loadings, report = gps.solve_single_unit(A, cfg)
            v1 = np.linalg.svd(A)[2][0]
            assert abs(loadings.values[:, 0] @ v1) >= 1 - 1e-8
            assert report.converged

    def test_monotone_history(self):
        rng = np.random.default_rng(18)
        for penalty in ("l1", "l0"):
            for _ in range(20):
                A = rng.standard_normal((5, 12))
                cfg = gps.SolverConfig(penalty=penalty, gamma=float(rng.uniform(0, 0.5)))
                _, report = gps.solve_single_unit(A, cfg)
                assert np.all(np.diff(report.objective_history) >= -1e-12)

    def test_sign_symmetry(self):
        rng = np.random.default_rng(19)
        A = rng.standard_normal((4, 9))
        x0 = rng.standard_normal(4)
        x0 /= np.linalg.norm(x0)
        for penalty in ("l1", "l0"):
            out = []
            for sign in (1.0, -1.0):
                cfg = gps.SolverConfig(penalty=penalty, gamma=0.2, init="user_supplied", x0=sign * x0, tol=1e-12)
                loadings, report = gps.solve_single_unit(A, cfg)
                out.append((loadings.values[:, 0], report.objective_history[-1]))
            (za, fa), (zb, fb) = out
            assert abs(fa - fb) <= 1e-10
            assert np.allclose(za, zb, atol=1e-9) or np.allclose(za, -zb, atol=1e-9)

    def test_m_one_multi_identical_to_single(self):
        rng = np.random.default_rng(23)
        A = rng.standard_normal((4, 7))
        cfg = gps.SolverConfig(penalty="l1", gamma=0.1, m=1)
        zs, rs = gps.solve_single_unit(A, cfg)
        zm, rm = gps.solve_multi_sequential(A, cfg)
        assert np.array_equal(zs.values, zm.values)
        assert rs.objective_history == rm.objective_history

    def test_zero_component_zero_fills_remainder(self):
        A = np.zeros((3, 2))
        A[0, 0] = 5.0
        A[1, 1] = 0.3
        loadings, report = gps.solve_multi_sequential(A, gps.SolverConfig(penalty="l1", gamma=1.0, m=2))
        assert loadings.nnz_per_component() == [1, 0]
        assert report.converged

    def test_deflate_matches_oracle(self):
        rng = np.random.default_rng(21)
        A = rng.standard_normal((4, 6))
        x = rng.standard_normal(4)
        x /= np.linalg.norm(x)
        out = gps.deflate(A, x)
        np.testing.assert_allclose(out.values, oracle.deflate(A, x), atol=1e-14)
        assert np.linalg.norm(x @ out.values) <= 1e-10

    def test_refine_and_restarts_p2(self):
        # acceptance criterion 2 in miniature: restarts + refine on p = 2
        rng = np.random.default_rng(102)
        theta = np.linspace(0, 2 * np.pi, 200_000, endpoint=False)
        circle = np.stack([np.cos(theta), np.sin(theta)])
        for _ in range(5):
            n = int(rng.integers(3, 12))
            A = rng.standard_normal((2, n))
            gamma = 0.3
            C = A.T @ circle
            grid = float((np.maximum(np.abs(C) - gamma, 0.0) ** 2).sum(axis=0).max())
            cfg = gps.SolverConfig(penalty="l1", gamma=gamma, tol=1e-12, max_iter=2000, restarts=n, refine=True)
            _, rep = gps.solve_single_unit(A, cfg)
            assert grid - rep.objective_history[-1] <= 1e-4


class TestLargeShapes:
    """Size-independent properties at BASELINE-like shapes (fp32 storage)."""

    def test_fused_sweep_vs_oracle_4096(self):
        rng = np.random.default_rng(5)
        p, n = 4096, 1 << 15
        A32 = rng.standard_normal((p, n), dtype=np.float32)
        A = gps.DataMatrix(np.asfortranarray(A32))
        x = rng.standard_normal(p)
        x /= np.linalg.norm(x)
        gamma = (0.1 * float(np.linalg.norm(A32.astype(np.float64), axis=0).max())) ** 2
        f, g, c, w, nnz = gps.fused_sweep(A, x, gamma, "l0", want_c=True, want_w=True)
        A64 = A32.astype(np.float64)
        c_ref = A64.T @ x
        np.testing.assert_allclose(c, c_ref, rtol=1e-11, atol=1e-11)
        w_ref = oracle.threshold(c_ref, gamma, "l0")
        assert_support_equal(w, w_ref, c_ref, gamma, "l0")
        np.testing.assert_allclose(g, A64 @ w_ref, rtol=1e-10, atol=1e-9)
        assert f == pytest.approx(oracle.su_objective(c_ref, gamma, "l0"), rel=1e-11)
        assert nnz == int(np.count_nonzero(w))

    def test_solve_deterministic_and_matches_oracle(self):
        rng = np.random.default_rng(6)
        p, n = 1000, 1 << 16
        A32 = rng.standard_normal((p, n), dtype=np.float32)
        A = gps.DataMatrix(np.asfortranarray(A32))
        gamma = 0.1 * float(A.norms.max())
        cfg = gps.SolverConfig(penalty="l1", gamma=gamma)
        z1, r1 = gps.solve_single_unit(A, cfg)
        z2, r2 = gps.solve_single_unit(A, cfg)
        assert r1.objective_history == r2.objective_history  # bitwise run-to-run
        assert np.array_equal(z1.values, z2.values)
        zo, ho, _, _ = oracle.su_solve(A32.astype(np.float64), gamma, "l1")
        assert len(ho) == len(r1.objective_history)
        np.testing.assert_allclose(r1.objective_history, ho, rtol=1e-9)
        np.testing.assert_allclose(z1.values[:, 0], zo, rtol=1e-7, atol=1e-9)


class TestWideP:
    """p beyond the fused kernels' register coverage (8192 fp32 / 4096 fp64)
    runs the two-pass wide fallback; results must match the oracle exactly
    as the fused path does."""

    @pytest.mark.parametrize("p,dtype", [(9000, np.float32), (4500, np.float64)])
    @pytest.mark.parametrize("penalty", ["l1", "l0"])
    def test_solve_matches_oracle(self, p, dtype, penalty):
        rng = np.random.default_rng(p)
        A32 = rng.standard_normal((p, 1500)).astype(np.float32)
        A64 = A32.astype(np.float64)
        gamma = 0.1 * float(np.linalg.norm(A64, axis=0).max())
        gamma = gamma if penalty == "l1" else gamma ** 2
        loadings, report = gps.solve_single_unit(gps.DataMatrix(A32.astype(dtype), dtype=dtype),
                                                 gps.SolverConfig(penalty=penalty, gamma=gamma))
        z, hist, conv, _ = oracle.su_solve(A64, gamma, penalty)
        assert report.iterations == len(hist) - 1
        np.testing.assert_allclose(report.objective_history, hist, rtol=1e-9)
        np.testing.assert_allclose(loadings.values[:, 0], z, rtol=1e-8, atol=1e-10)

    def test_kernel_seam_wide(self):
        rng = np.random.default_rng(1)
        A = rng.standard_normal((8300, 700))
        x = rng.standard_normal(8300)
        x /= np.linalg.norm(x)
        coef = rng.standard_normal(700)
        D = gps.DataMatrix(A.astype(np.float32))
        A32 = A.astype(np.float32).astype(np.float64)
        np.testing.assert_allclose(gps.par_matvec_t(D, x), A32.T @ x, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(gps.par_gram_apply(D, coef), A32 @ coef, rtol=1e-11, atol=1e-10)

    def test_block_wide_matches_oracle(self):
        rng = np.random.default_rng(2)
        A = rng.standard_normal((4200, 900))
        gamma = 0.1 * float(np.linalg.norm(A, axis=0).max())
        cfg = gps.SolverConfig(penalty="l1", mode="block", m=3, gamma=gamma)
        loadings, report = gps.solve_block(gps.DataMatrix(A), cfg)
        Z, hist, conv, _ = oracle.block_solve(A, 3, gamma, 1.0, "l1")
        assert report.iterations == len(hist) - 1
        np.testing.assert_allclose(report.objective_history, hist, rtol=1e-9)
        np.testing.assert_allclose(loadings.values, Z, rtol=1e-7, atol=1e-9)

"""The reference acceptance criteria that concern the hot path
(reference tests/test_acceptance.py), run on the device."""

from itertools import combinations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")

GAMMAS = (0.0, 0.01, 0.05, 0.3)


def test_criterion_01_monotone_ascent():
    # test_acceptance.py:52-82 (400 instances here instead of 1000)
    rng = np.random.default_rng(101)
    for _ in range(400):
        p, n = int(rng.integers(2, 31)), int(rng.integers(3, 101))
        A = rng.standard_normal((p, n))
        gamma = float(rng.choice(GAMMAS))
        m = 2 if min(p, n) >= 2 else 1
        for penalty in ("l1", "l0"):
            _, rep = gps.solve_single_unit(A, gps.SolverConfig(penalty=penalty, gamma=gamma, max_iter=300))
            assert np.all(np.diff(rep.objective_history) >= -1e-12)
            cfg = gps.SolverConfig(penalty=penalty, mode="block", m=m, gamma=gamma, init="random_orthonormal",
                                   seed=int(rng.integers(1 << 16)), max_iter=300)
            try:
                _, rep_b = gps.solve_block(A, cfg)
                history = rep_b.objective_history
            except gps.RankDeficiencyError as err:
                history = err.history
            assert np.all(np.diff(history) >= -1e-12)


def gapped_instance(rng, p, n, m):
    k = min(p, n)
    while True:
        s = np.sort(rng.uniform(0.5, 4.0, size=k))[::-1]
        if all(s[j] - s[j + 1] >= 0.1 for j in range(m)):
            break
    U = np.linalg.qr(rng.standard_normal((p, k)))[0]
    V = np.linalg.qr(rng.standard_normal((n, k)))[0]
    return U @ np.diag(s) @ V.T, V


def test_criterion_03_pca_equivalence_at_gamma_zero():
    # test_acceptance.py:124-159 (50 instances)
    rng = np.random.default_rng(103)
    for trial in range(50):
        A, V = gapped_instance(rng, int(rng.integers(4, 16)), int(rng.integers(4, 16)), m=2)
        penalty = "l1" if trial % 2 == 0 else "l0"
        loadings, _ = gps.solve_single_unit(A, gps.SolverConfig(penalty=penalty, gamma=0.0, tol=1e-14,
                                                                max_iter=20000))
        assert abs(loadings.values[:, 0] @ V[:, 0]) >= 1 - 1e-8
        cfg = gps.SolverConfig(penalty=penalty, mode="block", m=2, gamma=0.0, init="random_orthonormal",
                               seed=trial, tol=1e-14, max_iter=20000)
        loadings_b, _ = gps.solve_block(A, cfg)
        Q = np.linalg.qr(loadings_b.values)[0]
        cos = np.linalg.svd(Q.T @ V[:, :2], compute_uv=False)
        assert np.arccos(np.clip(cos.min(), 0.0, 1.0)) <= 1e-4


def enumerate_l0_supports(A, gamma):
    n = A.shape[1]
    sigma = A.T @ A
    best_val, best_z = 0.0, np.zeros(n)
    for size in range(1, n + 1):
        for S in combinations(range(n), size):
            w, V = np.linalg.eigh(sigma[np.ix_(S, S)])
            val = w[-1] - gamma * size
            if val > best_val:
                z = np.zeros(n)
                z[list(S)] = V[:, -1]
                best_val, best_z = val, z
    return best_val, best_z


def test_criterion_04_support_brute_force_l0():
    # test_acceptance.py:162-192: restarts + refine find the enumerated optimum
    rng = np.random.default_rng(104)
    for _ in range(10):
        A = rng.standard_normal((2, 4))
        gamma = float(rng.uniform(0.05, 0.8))
        cfg = gps.SolverConfig(penalty="l0", gamma=gamma, tol=1e-12, max_iter=2000, restarts=32, refine=True)
        loadings, rep = gps.solve_single_unit(A, cfg)
        val, z_star = enumerate_l0_supports(A, gamma)
        assert abs(rep.objective_history[-1] - val) <= 1e-6
        assert set(loadings.pattern[0].tolist()) == set(np.nonzero(np.abs(z_star) > 1e-12)[0].tolist())


def test_criterion_06_determinism():
    # test_acceptance.py:231-268 analogue: bitwise-identical kernel outputs run to run
    rng = np.random.default_rng(106)
    for _ in range(5):
        A = gps.DataMatrix(rng.standard_normal((64, 4096)))
        x = rng.standard_normal(64)
        z = rng.standard_normal(4096)
        c = gps.par_matvec_t(A, x)
        for fn, args in ((gps.par_matvec_t, (A, x)), (gps.par_gram_apply, (A, z)),
                         (gps.par_threshold_accumulate, (A, c, 0.05, "l1")),
                         (gps.par_threshold_accumulate, (A, c, 0.05, "l0"))):
            outs = [fn(*args, gps.KernelPlan(workers=w)) for w in (1, 2, 4, 8)]
            for other in outs[1:]:
                assert np.array_equal(outs[0], other)


def test_criterion_10_gamma_monotone_support():
    # test_acceptance.py:350-364 (300 triples)
    rng = np.random.default_rng(110)
    for _ in range(300):
        p, n = int(rng.integers(2, 12)), int(rng.integers(3, 30))
        A = gps.DataMatrix(rng.standard_normal((p, n)))
        x = rng.standard_normal(p)
        x /= np.linalg.norm(x)
        lo_g = float(rng.uniform(0.0, 1.0))
        hi_g = lo_g + float(rng.uniform(0.0, 1.0))
        for recover in (gps.recover_pattern_sl1, gps.recover_pattern_sl0):
            lo = set(np.nonzero(recover(A, x, lo_g))[0].tolist())
            hi = set(np.nonzero(recover(A, x, hi_g))[0].tolist())
            assert hi <= lo

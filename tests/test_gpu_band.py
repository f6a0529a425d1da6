"""The near-threshold log (north_star: support entries within 1e-6 gamma of
the threshold are logged; RunReport.near_threshold).

Fixed-point instances make the final sweep's correlations known exactly:
every column is a multiple of a coordinate vector, so x = e_1 (single unit)
or X = [e_1 e_2] (block) is a fixed point of the power map, and the planted
columns sit at relative distances 1e-7 (inside the band, on both sides of
the threshold) and 1e-4 (outside) from it.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")


def _su_matrix(penalty, gamma):
    # c_i = first coordinate; threshold on |c| (l1) or c^2 (l0)
    t = gamma if penalty == "l1" else np.sqrt(gamma)
    rows = [5.0 * t, -3.0 * t, 2.0 * t,  # active, far from the threshold
            0.2 * t, -0.5 * t,            # inactive, far
            t * (1 + 1e-7), -t * (1 - 1e-7),  # in band: active / inactive
            t * (1 + 1e-4), t * (1 - 1e-4)]   # outside the band
    A = np.zeros((3, len(rows)))
    A[0] = rows
    return A


@pytest.mark.parametrize("penalty", ["l1", "l0"])
def test_su_band_exact(penalty):
    gamma = 0.7
    band_scale = 1e-6 * gamma
    A = _su_matrix(penalty, gamma)
    x0 = np.array([1.0, 0.0, 0.0])
    cfg = gps.SolverConfig(penalty=penalty, gamma=gamma, init="user_supplied", x0=x0)
    loadings, report = gps.solve_single_unit(gps.DataMatrix(A), cfg)
    got = set(report.near_threshold[0].tolist())
    c = A[0]
    dist = np.abs(np.abs(c) - gamma) if penalty == "l1" else np.abs(c * c - gamma)
    want = set(np.flatnonzero(dist <= band_scale).tolist())
    assert want == {5, 6}
    assert got == want
    assert report.near_threshold_total == 2
    assert set(loadings.pattern[0].tolist()) == {0, 1, 2, 5, 7}


def test_block_band_exact_mu_scaled():
    gamma = np.array([0.5, 0.8])
    mu = np.array([1.0, 0.6])
    t1, t2 = gamma[0] / mu[0], gamma[1] / mu[1]   # l1 thresholds on |c| per component
    cols = []
    for v in (4 * t1, -2 * t1, t1 * (1 + 1e-7), t1 * (1 - 1e-7), t1 * (1 + 1e-4)):
        cols.append([v, 0, 0, 0])
    for v in (3 * t2, t2 * (1 - 1e-7), -t2 * (1 + 1e-7), t2 * 0.1):
        cols.append([0, v, 0, 0])
    A = np.array(cols).T
    X0 = np.eye(4)[:, :2]
    cfg = gps.SolverConfig(penalty="l1", mode="block", m=2, gamma=gamma, mu=mu, init="user_supplied", x0=X0)
    loadings, report = gps.solve_block(gps.DataMatrix(A), cfg)
    assert set(report.near_threshold[0].tolist()) == {2, 3}
    assert set(report.near_threshold[1].tolist()) == {6, 7}
    assert report.near_threshold_total == 4
    assert max(report.stiefel_errors) <= 1e-15


def test_gamma_zero_has_no_band():
    A = np.zeros((3, 5))
    A[0, :3] = [1.0, 0.0, -2.0]
    cfg = gps.SolverConfig(penalty="l0", gamma=0.0, init="user_supplied", x0=np.array([1.0, 0, 0]))
    _, report = gps.solve_single_unit(gps.DataMatrix(A), cfg)
    assert report.near_threshold_total == 0

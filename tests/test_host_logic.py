"""Host-side logic that needs no GPU: config validation, value types,
threshold rule, partitioning."""

import numpy as np
import pytest

import paper_1312_6182_b200 as gps
from paper_1312_6182_b200.distributed import column_partition


class TestSolverConfig:
    def test_broadcasts_gamma_mu(self):
        cfg = gps.SolverConfig(m=3, gamma=0.5, mu=2.0)
        assert cfg.gamma.tolist() == [0.5] * 3 and cfg.mu.tolist() == [2.0] * 3
        with pytest.raises(ValueError):
            cfg.gamma[0] = 1.0

    @pytest.mark.parametrize("kw", [dict(penalty="l2"), dict(mode="x"), dict(init="y"), dict(m=0),
                                    dict(restarts=0), dict(tol=0.0), dict(max_iter=0), dict(gamma=-1.0),
                                    dict(mu=0.0), dict(init="user_supplied"), dict(m=2, gamma=[1.0, 2.0, 3.0])])
    def test_rejects(self, kw):
        with pytest.raises(ValueError):
            gps.SolverConfig(**kw)


class TestValueTypes:
    def test_sparse_loadings_pattern_and_norm_check(self):
        z = gps.SparseLoadings([0.0, 0.6, 0.0, 0.8])
        assert z.nnz_per_component() == [2]
        assert z.pattern[0].tolist() == [1, 3]
        with pytest.raises(ValueError):
            gps.SparseLoadings([1.0, 1.0])
        with pytest.raises(AttributeError):
            z.m = 3

    def test_stiefel_point(self):
        gps.StiefelPoint(np.eye(3)[:, :2])
        with pytest.raises(ValueError):
            gps.StiefelPoint(np.ones((3, 2)))
        with pytest.raises(ValueError):
            gps.StiefelPoint(np.eye(2, 3))

    def test_kernel_plan(self):
        with pytest.raises(ValueError):
            gps.KernelPlan(workers=0)
        with pytest.raises(ValueError):
            gps.KernelPlan(reduction="left_to_right")

    def test_threshold_weights(self):
        c = np.array([-2.0, -0.1, 0.0, 0.1, 2.0])
        assert np.allclose(gps.threshold_weights(c, 0.5, "l1"), [-1.5, 0, 0, 0, 1.5])
        assert np.allclose(gps.threshold_weights(c, 0.5, "l0"), [-2.0, 0, 0, 0, 2.0])
        assert gps.threshold_weights(np.array([1.0]), 1.0, "l0").tolist() == [0.0]

    def test_power_step(self):
        st = gps.SingleUnitState(x=np.array([1.0, 0.0]), objective=0.0, iteration=0)
        nxt, fixed = gps.power_step(st, np.array([3.0, 4.0]))
        assert not fixed and np.allclose(nxt.x, [0.6, 0.8]) and nxt.iteration == 1
        same, fixed = gps.power_step(st, np.zeros(2))
        assert fixed and same is st


@pytest.mark.parametrize("n,world", [(10, 1), (10, 3), (1 << 20, 8), (7, 7)])
def test_column_partition(n, world):
    parts = column_partition(n, world)
    assert parts[0][0] == 0 and sum(k for _, k in parts) == n
    for (o1, k1), (o2, _) in zip(parts, parts[1:]):
        assert o1 + k1 == o2
    assert max(k for _, k in parts) - min(k for _, k in parts) <= 1


def test_decode_band_entries():
    """Near-threshold entries are col * 64 + component (csrc/common.cuh
    BandLog); decode_band groups them per component, sorted and unique,
    shifted by the shard offset."""
    from paper_1312_6182_b200.core import decode_band

    entries = np.array([5 * 64 + 1, 2 * 64 + 0, 9 * 64 + 1, 2 * 64 + 0, 7 * 64 + 3], dtype=np.int64)
    out = decode_band(entries, 4, offset=100)
    assert [o.tolist() for o in out] == [[102], [105, 109], [], [107]]
    assert [o.tolist() for o in decode_band(np.zeros(0, dtype=np.int64), 2)] == [[], []]

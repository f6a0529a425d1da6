"""The peer-memory all-reduce of the sharded loops (csrc/px_kernels.cuh,
gps_px_*).  One GPU cannot run ranks that wait on each other as separate
launches, so the multi-rank protocol (push into every rank's symmetric
buffer, release/acquire epoch flags, parity-double-buffered slots, rank-order
sum) is run as ONE cooperative kernel over all emulated ranks' buffers on
the device, for several rounds (epochs of both parities); the result must be
bitwise the rank-order sum on every rank.  The real per-rank kernel is run
at world size 1 (its own push and flags)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")
from paper_1312_6182_b200 import _native  # noqa: E402


def rank_order_sum(vecs):
    s = vecs[0].copy()
    for v in vecs[1:]:
        s = s + v
    return s


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("count", [5, 4100, 3 * 4096 + 7])
def test_emulated_ranks_sum_in_rank_order(world, count):
    rng = np.random.default_rng(world * 1000 + count)
    vin = rng.standard_normal((world, count)) * np.logspace(0, 8, world)[:, None]
    rounds = 3
    out = np.empty((rounds, world, count))
    ctx = _native.context(0)
    _native.check(_native.lib().gps_px_emulate(ctx.handle, world, count, rounds, _native.dptr(np.ascontiguousarray(vin)),
                                               out.ctypes.data_as(_native._dp)))
    for k in range(rounds):
        ref = rank_order_sum([vin[r] * (k + 1) for r in range(world)])
        for r in range(world):
            assert np.array_equal(out[k, r], ref), (k, r)


def test_world_one_kernel_repeats():
    import torch

    ctx = _native.context(0)
    L = _native.lib()
    h = _native._vp()
    _native.check(L.gps_px_create(ctx.handle, 1, 0, 5000, _native.C.byref(h)))
    try:
        size = L.gps_px_handle_size()
        assert size >= 64
        t = torch.arange(5000, dtype=torch.float64, device="cuda:0")
        torch.cuda.synchronize()
        for _ in range(5):  # epochs 1..5, both parities
            _native.check(L.gps_px_allreduce(h, _native._vp(t.data_ptr())))
        ctx.sync()
        assert torch.equal(t.cpu(), torch.arange(5000, dtype=torch.float64))
    finally:
        L.gps_px_destroy(h)


def test_bad_arguments():
    ctx = _native.context(0)
    h = _native._vp()
    with pytest.raises(NotImplementedError):
        _native.check(_native.lib().gps_px_create(ctx.handle, 9, 0, 10, _native.C.byref(h)))
    with pytest.raises(ValueError):
        _native.check(_native.lib().gps_px_create(ctx.handle, 2, 2, 10, _native.C.byref(h)))
    _native.check(_native.lib().gps_px_create(ctx.handle, 2, 0, 10, _native.C.byref(h)))
    try:
        buf = np.zeros(10)
        with pytest.raises(ValueError):  # peer 1 not opened
            _native.check(_native.lib().gps_px_allreduce(h, buf.ctypes.data_as(_native._vp)))
    finally:
        _native.lib().gps_px_destroy(h)

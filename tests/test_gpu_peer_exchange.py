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


def k2_reference(pg, ps, rows):
    """su_reduce_kernel's fixed order: 8 contiguous slices of the partials per
    row summed sequentially, then the slices in order; scalars: lane-strided
    (32 lanes) sequential sums combined by the xor butterfly."""
    nparts = pg.shape[0]
    out = np.empty(rows + 4)
    slices = []
    for sl in range(8):
        b0, b1 = nparts * sl // 8, nparts * (sl + 1) // 8
        t = np.zeros(rows)
        for b in range(b0, b1):
            t = t + pg[b]
        slices.append(t)
    u = slices[0].copy()
    for k in range(1, 8):
        u = u + slices[k]
    out[:rows] = u
    ns = ps.shape[0]
    for k in range(4):
        lanes = np.zeros(32)
        for lane in range(32):
            t = 0.0
            for b in range(lane, ns, 32):
                t = t + ps[b, k]
            lanes[lane] = t
        o = 16
        while o:
            lanes = lanes + lanes[np.arange(32) ^ o]
            o >>= 1
        out[rows + k] = lanes[0]
    return out


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("rows,nparts,nparts_s", [(4096, 148, 148), (640, 32, 296), (3 * 4096 + 96, 32, 5)])
def test_fused_reduce_exchange_emulated(world, rows, nparts, nparts_s):
    rng = np.random.default_rng(rows + world)
    pg = rng.standard_normal((world, nparts, rows))
    ps = rng.standard_normal((world, nparts_s, 4))
    rounds = 2
    out = np.empty((rounds, world, rows + 4))
    ctx = _native.context(0)
    _native.check(_native.lib().gps_px_emulate_reduce(ctx.handle, world, rows, nparts, nparts_s, rounds,
                                                      _native.dptr(np.ascontiguousarray(pg)),
                                                      _native.dptr(np.ascontiguousarray(ps)),
                                                      out.ctypes.data_as(_native._dp)))
    for k in range(rounds):
        per_rank = [k2_reference(pg[r] * (k + 1), ps[r] * (k + 1), rows) for r in range(world)]
        ref = rank_order_sum(per_rank)
        for r in range(world):
            assert np.array_equal(out[k, r], ref), (k, r)


def test_fused_reduce_world_one_solve_matches():
    """A world-size-1 peer exchange attached to a single-unit loop: the fused
    K2 must reproduce the unfused solve bitwise."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((300, 2001)).astype(np.float32)
    D = gps.DataMatrix(A)
    gamma = 0.1 * float(np.asarray(D.norms).max())
    ref_loop = gps.single_unit.PowerLoop(D, "l1", gamma, 1e-6, 200)
    x0 = D.column(int(np.argmax(D.norms))) / float(np.max(D.norms))
    x_ref, h_ref, c_ref, w_ref = ref_loop.run(x0)
    L = _native.lib()
    ctx = D.context
    h = _native._vp()
    _native.check(L.gps_px_create(ctx.handle, 1, 0, 320 + 4, _native.C.byref(h)))  # ld = roundup(300, 32)
    try:
        loop = gps.single_unit.PowerLoop(D, "l1", gamma, 1e-6, 200)
        _native.check(L.gps_su_attach_px(loop.handle, h))
        x, hist, conv, w = loop.run(x0)
        assert hist == h_ref and np.array_equal(w, w_ref) and np.array_equal(x, x_ref)
        del loop
    finally:
        L.gps_px_destroy(h)


def test_fused_step_world_one_with_deflation():
    """The power step fused into the exchange kernel's last CTA (one launch
    fewer per iteration) with implicit deflation active: bitwise equal to
    the separate K3."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((300, 3001)).astype(np.float32)
    D = gps.DataMatrix(A)
    gamma = 0.05 * float(np.asarray(D.norms).max())
    X = np.linalg.qr(rng.standard_normal((300, 2)))[0]
    x0 = rng.standard_normal(300)
    x0 -= X @ (X.T @ x0)
    x0 /= np.linalg.norm(x0)
    ref_loop = gps.single_unit.PowerLoop(D, "l1", gamma, 1e-8, 300)
    ref_loop.set_deflation(X)
    x_ref, h_ref, _, w_ref = ref_loop.run(x0)
    L = _native.lib()
    h = _native._vp()
    _native.check(L.gps_px_create(D.context.handle, 1, 0, 320 + 4, _native.C.byref(h)))
    try:
        loop = gps.single_unit.PowerLoop(D, "l1", gamma, 1e-8, 300)
        loop.set_deflation(X)
        _native.check(L.gps_su_attach_px(loop.handle, h))
        assert L.gps_su_launches_per_iter(loop.handle) == 2
        x, hist, _, w = loop.run(x0)
        assert hist == h_ref and np.array_equal(w, w_ref) and np.array_equal(x, x_ref)
        del loop
    finally:
        L.gps_px_destroy(h)


def test_exchange_wait_is_bounded():
    """A rank whose peers never arrive times out (error flag) instead of
    spinning forever (px_gather's globaltimer deadline)."""
    import time

    ctx = _native.context()
    err = _native.C.c_int(0)
    t0 = time.perf_counter()
    _native.check(_native.lib().gps_px_emulate_timeout(ctx.handle, 2, 5000, 0.2, _native.C.byref(err)))
    assert err.value == 1
    assert time.perf_counter() - t0 < 30

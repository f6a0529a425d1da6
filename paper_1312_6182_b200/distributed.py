"""Column-sharded GP-SPCA across GPUs (one process per GPU).

SURVEY §8(e): A is split by columns -- rank r owns the contiguous block
[offset_r, offset_r + n_r) -- so every column's correlation, threshold,
objective term and rank-1 update stay local.  The only exchange per power
iteration is ONE all-reduce (sum) of the exchange vector
[g (ld) | f | nnz | sum w^2 | 0] produced by each rank's sweep + local
reduction; every rank then runs the identical step kernel on identical
data, so no second exchange is needed.  Per solve: a max all-reduce for the
activation limit, an all-gather of (max norm, global index) for the
max-norm-column start plus a broadcast of the winning column, and a sum
all-reduce of ||w||^2 for the recovery normalisation.

The per-iteration all-reduce runs on the devices inside the loop's own
cross-CTA reduction kernel over NVLink peer memory (PeerExchange attached to
the loop, gps_px_*: every rank's K2 stores its reduced exchange vector into
every peer's symmetric buffer, then sums the ranks' vectors in rank order)
when every GPU pair has peer access;
otherwise (or with GPSPCA_EXCHANGE=nccl) it is a torch.distributed
all-reduce.  The per-solve collectives and the handle exchange are
torch.distributed (NCCL on GPUs; gloo in the CPU tests).  The loop driver is
written against a small "shard loop" protocol so the CPU tests can drive it
with gloo and a test-side loop.
"""

import os

import time

import numpy as np

from . import _native
from .core import RunReport, SparseLoadings
from .block import BlockLoop, RankDeficiencyError, _as_stiefel_values
from .core import StiefelPoint
from .single_unit import PowerLoop, _check_unit, _random_unit


def column_partition(n, world):
    """Contiguous, balanced column blocks: [(offset, count)] per rank."""
    if world < 1 or n < world:
        raise ValueError(f"cannot split {n} columns over {world} ranks")
    bounds = [n * r // world for r in range(world + 1)]
    return [(bounds[r], bounds[r + 1] - bounds[r]) for r in range(world)]


class DeviceShardLoop:
    """PowerLoop on this rank's shard with a torch-owned exchange buffer
    (so torch.distributed can all-reduce it in place on the same stream)."""

    def __init__(self, A_local, penalty, gamma, tol, max_iter):
        import torch

        self.A = A_local
        self.A_context = A_local.context
        self.loop = PowerLoop(A_local, penalty, gamma, tol, max_iter)
        n_exch = _native.C.c_int64()
        _native.check(_native.lib().gps_su_exchange(self.loop.handle, None, _native.C.byref(n_exch)))
        dev = torch.device("cuda", A_local.context.device)
        self.buf = torch.zeros(n_exch.value, dtype=torch.float64, device=dev)
        _native.check(_native.lib().gps_su_set_exchange(self.loop.handle, _native.C.c_void_p(self.buf.data_ptr())))
        stream = torch.cuda.current_stream(dev)
        if stream.cuda_stream == 0:  # the legacy default stream cannot be captured; use a side stream
            stream = torch.cuda.Stream(dev)
            torch.cuda.set_stream(stream)
        A_local.context.set_stream(stream.cuda_stream)

    def start(self, x0):
        self.loop.start(x0)

    def attach_px(self, comm, device):
        px = PeerExchange(self.A_context, comm, self.buf.numel())  # ld + 4
        if not px_self_test(px, comm, device, self.buf.numel()):
            return False
        self.px = px
        _native.check(_native.lib().gps_su_attach_px(self.loop.handle, self.px.handle), "gps_su_attach_px")
        return True

    def enqueue_sweep(self):
        _native.check(_native.lib().gps_su_enqueue_sweep(self.loop.handle))

    def exchange(self):
        return self.buf

    def enqueue_step(self):
        _native.check(_native.lib().gps_su_enqueue_step(self.loop.handle))

    def poll(self):
        d, it, cv = _native.C.c_int(), _native.C.c_int(), _native.C.c_int()
        _native.check(_native.lib().gps_su_poll(self.loop.handle, _native.C.byref(d), _native.C.byref(it),
                                                _native.C.byref(cv)))
        return bool(d.value), it.value, bool(cv.value)

    def result(self):
        return self.loop.result()


class PeerExchange:
    """Sum all-reduce of a device float64 vector of fixed length over NVLink
    peer memory (gps_px_*), one kernel per rank; identical result, summed in
    rank order, on every rank.  Collective construction: every rank of the
    group builds it with the same count."""

    def __init__(self, context, comm, count):
        import torch.distributed as dist

        L = _native.lib()
        self.count = int(count)
        self.handle = None
        # Every rank reaches the one collective below whatever fails locally
        # (a rank raising before it would leave its peers blocked in it);
        # failures are recorded in self.ok, which px_self_test agrees on.
        self.ok = True
        mine = None
        try:
            h = _native._vp()
            _native.check(L.gps_px_create(context.handle, comm.world, comm.rank, self.count, _native.C.byref(h)),
                          "gps_px_create")
            self.handle = h
            size = L.gps_px_handle_size()
            buf = (_native.C.c_char * size)()
            _native.check(L.gps_px_ipc_handle(h, buf), "gps_px_ipc_handle")
            mine = bytes(buf)
        except Exception:  # noqa: BLE001 -- reported through self.ok
            self.ok = False
        handles = [None] * comm.world
        dist.all_gather_object(handles, mine, group=comm.group)
        if self.ok and all(hb is not None for hb in handles):
            try:
                size = L.gps_px_handle_size()
                for peer, hb in enumerate(handles):
                    _native.check(L.gps_px_open(self.handle, peer, (_native.C.c_char * size).from_buffer_copy(hb)),
                                  "gps_px_open")
            except Exception:  # noqa: BLE001 -- reported through self.ok
                self.ok = False
        else:
            self.ok = False

    def all_reduce(self, t):
        assert self.ok, "peer exchange not usable on this rank"
        assert t.numel() == self.count and t.dtype.is_floating_point and t.element_size() == 8
        _native.check(_native.lib().gps_px_allreduce(self.handle, _native._vp(t.data_ptr())), "gps_px_allreduce")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            _native.lib().gps_px_destroy(h)
            self.handle = None


def peer_exchange_available(comm, device):
    """Peer-memory all-reduce applies: every rank on its OWN CUDA device (two
    ranks spinning on one GPU could wait on each other forever), world in
    [2, 8], every pair of those devices with peer access, and not disabled by
    GPSPCA_EXCHANGE=nccl.  Decided identically on every rank."""
    import torch

    if os.environ.get("GPSPCA_EXCHANGE", "").lower() == "nccl" or not 2 <= comm.world <= 8:
        return False
    dev = device.index if isinstance(device, torch.device) and device.type == "cuda" else None
    devs = [None] * comm.world
    comm.dist.all_gather_object(devs, dev, group=comm.group)
    if any(d is None for d in devs) or len(set(devs)) != comm.world:
        return False
    return all(torch.cuda.can_device_access_peer(a, b) for a in devs for b in devs if a != b)


SELF_TEST_TIMEOUT_S = 5.0


def px_self_test(px, comm, device, count):
    """Collective check of a freshly opened peer exchange: one standalone
    peer-memory all-reduce of a seeded vector against the torch.distributed
    all-reduce (NCCL) of the same vector.  Returns True on every rank only
    if every rank's result agrees (1e-12; the rank-order and NCCL summation
    orders differ in rounding) and no rank raised -- callers fall back to
    the torch.distributed exchange otherwise, so a peer path that cannot run
    on a given machine costs speed, never results."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(1234 + comm.rank)
    v = torch.randn(count, dtype=torch.float64, device=device, generator=g)
    ref = v.clone()
    comm.dist.all_reduce(ref, op=comm.dist.ReduceOp.SUM, group=comm.group)
    # a rank whose construction failed must not launch: its peers' pushes
    # would wait on it until the timeout (they agree below and fall back)
    flag0 = torch.tensor([1 if getattr(px, "ok", True) else 0], dtype=torch.int32, device=device)
    comm.dist.all_reduce(flag0, op=comm.dist.ReduceOp.MIN, group=comm.group)
    if not bool(flag0.item()):
        return False
    try:
        # a peer path that cannot deliver (flags never visible) times out in
        # seconds here rather than the loop's 60 s bound
        handle = getattr(px, "handle", None)
        if handle is not None:
            _native.lib().gps_px_set_timeout(handle, SELF_TEST_TIMEOUT_S)
        px.all_reduce(v)
        torch.cuda.synchronize(device)
        ok = bool(torch.allclose(v, ref, rtol=1e-12, atol=1e-12))
        if handle is not None:
            err = _native.C.c_int(0)
            _native.check(_native.lib().gps_px_error(handle, _native.C.byref(err)), "gps_px_error")
            ok = ok and err.value == 0
            _native.lib().gps_px_set_timeout(handle, float(os.environ.get("GPSPCA_PX_TIMEOUT_S", "60") or 60))
    except Exception:  # noqa: BLE001 -- any failure means "do not use the peer path"
        ok = False
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
    comm.dist.all_reduce(flag, op=comm.dist.ReduceOp.MIN, group=comm.group)
    return bool(flag.item())


def loop_all_reduce(loop, comm, device):
    """The per-iteration exchange of a device shard loop.  With peer access
    between every rank's GPU, a PeerExchange is attached to the loop and the
    loop's own cross-CTA reduction kernel (K2) performs the all-reduce --
    compute and collective in one kernel -- so the returned callable does
    nothing; otherwise the torch.distributed all-reduce."""
    if hasattr(loop, "attach_px") and peer_exchange_available(comm, device):
        if loop.attach_px(comm, device):
            return lambda t: None
    return comm.all_reduce_sum


def run_sharded_loop(loop, all_reduce, poll_every=8, max_iter=1000):
    """Drive a started shard loop to its stopping rule: per iteration sweep
    -> all_reduce(exchange) -> step; poll the control block every chunk."""
    for _ in range(max_iter // poll_every + 2):
        for _ in range(poll_every):
            loop.enqueue_sweep()
            all_reduce(loop.exchange())
            loop.enqueue_step()
        done, _, _ = loop.poll()
        if done:
            return loop.result()
    raise RuntimeError("sharded power loop did not stop within max_iter")


class Comm:
    """The four collectives the sharded solve needs, over torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def _host(self, arr, like=None):
        import torch

        return torch.as_tensor(np.asarray(arr, dtype=np.float64), device=like if like is not None else "cpu")

    def max_scalar(self, v, device="cpu"):
        import torch

        t = torch.tensor([float(v)], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def sum_scalar(self, v, device="cpu"):
        import torch

        t = torch.tensor([float(v)], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return float(t.item())

    def all_gather_vec(self, v, device="cpu"):
        import torch

        t = torch.as_tensor(np.asarray(v, dtype=np.float64)).to(device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    def broadcast_vec(self, v, src, size, device="cpu"):
        import torch

        t = (torch.as_tensor(np.asarray(v, dtype=np.float64)) if v is not None
             else torch.empty(size, dtype=torch.float64)).to(device)
        self.dist.broadcast(t, src=src, group=self.group)
        return t.cpu().numpy()


def global_max_norm_start(norms_local, offset, column_fn, comm, p, device="cpu"):
    """max_norm_column init across shards (single_unit.py:151-153): the
    largest norm wins, ties go to the lowest GLOBAL index."""
    i_loc = int(np.argmax(norms_local))
    cand = comm.all_gather_vec([norms_local[i_loc], offset + i_loc], device)
    best_val = max(c[0] for c in cand)
    owner = min(r for r, c in enumerate(cand) if c[0] == best_val and
                c[1] == min(cc[1] for cc in cand if cc[0] == best_val))
    col = column_fn(int(cand[owner][1]) - offset) if comm.rank == owner else None
    col = comm.broadcast_vec(col, owner, p, device)
    return col / best_val, best_val


def solve_single_unit_sharded(A_local, config, offset, n_global, comm=None, loop_factory=None,
                              device="cpu", poll_every=8):
    """Sharded drop-in for solve_single_unit (single_unit.py:184-210).

    A_local: this rank's DataMatrix (or a test stand-in exposing .norms,
    .column(i), .p, .n).  Returns (SparseLoadings over ALL n_global columns,
    RunReport) on every rank."""
    comm = comm or Comm()
    if config.mode != "single_unit" or config.m != 1:
        raise ValueError("solve_single_unit_sharded handles mode='single_unit', m=1")
    if config.refine or config.restarts != 1:
        raise NotImplementedError("restarts/refine are single-device features")
    gamma = float(config.gamma[0])
    start = time.perf_counter()
    top = comm.max_scalar(float(np.max(A_local.norms)), device)
    limit = top if config.penalty == "l1" else top * top
    if gamma >= limit:
        z = np.zeros(n_global)
        loadings = SparseLoadings(z)
        return loadings, RunReport([0.0], 0, time.perf_counter() - start, loadings.nnz_per_component(), True,
                                   [[0.0]])
    if config.init == "user_supplied":
        x0 = _check_unit(config.x0, A_local.p)
    elif config.init == "random_orthonormal":
        x0 = _random_unit(np.random.default_rng(config.seed), A_local.p)
    else:
        x0, _ = global_max_norm_start(A_local.norms, offset, A_local.column, comm, A_local.p, device)
    factory = loop_factory or DeviceShardLoop
    loop = factory(A_local, config.penalty, gamma, config.tol, config.max_iter)
    loop.start(x0)
    x, history, converged, w_local = run_sharded_loop(loop, loop_all_reduce(loop, comm, device), poll_every,
                                                      config.max_iter)
    s2 = comm.sum_scalar(float(w_local @ w_local), device)
    z_local = w_local / np.sqrt(s2) if s2 > 0 else w_local
    z = _gather_ragged(comm, z_local, offset, n_global, device)
    loadings = SparseLoadings(z)
    return loadings, RunReport(history, len(history) - 1, time.perf_counter() - start,
                               loadings.nnz_per_component(), converged, [history])


def _gather_ragged(comm, z_local, offset, n_global, device):
    """All-gather for unequal shards: pad to the largest shard."""
    kmax = int(comm.max_scalar(len(z_local), device))
    buf = np.zeros(kmax + 2)
    buf[0], buf[1] = offset, len(z_local)
    buf[2:2 + len(z_local)] = z_local
    z = np.zeros(n_global)
    for part in comm.all_gather_vec(buf, device):
        o, k = int(part[0]), int(part[1])
        z[o:o + k] = part[2:2 + k]
    return z


# ------------------------------------------------------------------ block


class DeviceBlockShardLoop:
    """BlockLoop on this rank's shard with a torch-owned exchange buffer
    ([groups][MG*ld + 4]: per-group G partials, f, nnz)."""

    def __init__(self, A_local, penalty, m, gamma, mu, tol, max_iter):
        import torch

        self.loop = BlockLoop(A_local, penalty, m, gamma, mu, tol, max_iter)
        self.A_context = A_local.context
        n_exch = _native.C.c_int64()
        _native.check(_native.lib().gps_bk_exchange(self.loop.handle, None, _native.C.byref(n_exch)))
        dev = torch.device("cuda", A_local.context.device)
        self.buf = torch.zeros(n_exch.value, dtype=torch.float64, device=dev)
        _native.check(_native.lib().gps_bk_set_exchange(self.loop.handle, _native.C.c_void_p(self.buf.data_ptr())))
        stream = torch.cuda.current_stream(dev)
        if stream.cuda_stream == 0:
            stream = torch.cuda.Stream(dev)
            torch.cuda.set_stream(stream)
        A_local.context.set_stream(stream.cuda_stream)

    def start(self, M, orthonormalize):
        (self.loop.start_qr if orthonormalize else self.loop.start_user)(M)

    def attach_px(self, comm, device):
        stride = _native.C.c_int64()
        _native.check(_native.lib().gps_bk_exchange_stride(self.loop.handle, _native.C.byref(stride)))
        px = PeerExchange(self.A_context, comm, stride.value)  # one group's exchange vector
        if not px_self_test(px, comm, device, stride.value):
            return False
        self.px = px
        _native.check(_native.lib().gps_bk_attach_px(self.loop.handle, self.px.handle), "gps_bk_attach_px")
        return True

    def enqueue_sweep(self):
        _native.check(_native.lib().gps_bk_enqueue_sweep(self.loop.handle))

    def exchange(self):
        return self.buf

    def enqueue_step(self):
        _native.check(_native.lib().gps_bk_enqueue_step(self.loop.handle))

    def poll(self):
        d, it, cv = _native.C.c_int(), _native.C.c_int(), _native.C.c_int()
        _native.check(_native.lib().gps_bk_poll(self.loop.handle, _native.C.byref(d), _native.C.byref(it),
                                                _native.C.byref(cv)))
        return bool(d.value), it.value, bool(cv.value)

    def result(self):
        return self.loop.result()


def global_top_m_columns(norms_local, offset, column_fn, comm, m, p, device="cpu"):
    """block.py:157-158 across shards: the m largest norms, ties to the lowest
    GLOBAL index (stable argsort of -norms); returns M (p x m), identical on
    every rank (owners fill their columns, one sum all-reduce)."""
    k = min(m, len(norms_local))
    loc = np.argsort(-np.asarray(norms_local), kind="stable")[:k]
    cand = np.full(2 * m, -1.0)
    cand[:k] = np.asarray(norms_local)[loc]
    cand[m:m + k] = offset + loc
    allc = comm.all_gather_vec(cand, device)
    pairs = [(c[i], int(c[m + i])) for c in allc for i in range(m) if c[m + i] >= 0]
    pairs.sort(key=lambda t: (-t[0], t[1]))
    chosen = [g for _, g in pairs[:m]]
    M = np.zeros((p, m))
    n_local = len(norms_local)
    for j, g in enumerate(chosen):
        if offset <= g < offset + n_local:
            M[:, j] = column_fn(g - offset)
    import torch

    t = torch.as_tensor(M.ravel(order="F")).to(device)
    comm.dist.all_reduce(t, op=comm.dist.ReduceOp.SUM, group=comm.group)
    return t.cpu().numpy().reshape((p, m), order="F"), chosen


def solve_block_sharded(A_local, config, offset, n_global, comm=None, loop_factory=None, device="cpu",
                        poll_every=8):
    """Sharded drop-in for solve_block (block.py:190-235).  Returns
    (SparseLoadings over all n_global columns, RunReport) on every rank and
    raises RankDeficiencyError identically on every rank."""
    comm = comm or Comm()
    if config.mode != "block":
        raise ValueError("solve_block requires mode='block'")
    p, m = A_local.p, config.m
    if not 1 <= m <= min(p, n_global):
        raise ValueError(f"need 1 <= m <= min(p, n) = {min(p, n_global)}, got m={m}")
    start = time.perf_counter()
    if config.init == "random_orthonormal":
        M, ortho = np.random.default_rng(config.seed).standard_normal((p, m)), True
    elif config.init == "max_norm_column":
        M, _ = global_top_m_columns(A_local.norms, offset, A_local.column, comm, m, p, device)
        ortho = True
    else:
        M = StiefelPoint(_as_stiefel_values(config.x0, p, m)).values
        ortho = False
    factory = loop_factory or DeviceBlockShardLoop
    loop = factory(A_local, config.penalty, m, config.gamma, config.mu, config.tol, config.max_iter)
    loop.start(M, ortho)
    X, history, converged, W_local, rank_fail, rank = run_sharded_loop(loop, loop_all_reduce(loop, comm, device),
                                                                      poll_every, config.max_iter)
    if rank_fail:
        err = RankDeficiencyError(rank, m, iteration=len(history) - 1)
        err.history = history
        raise err
    StiefelPoint(X)  # block.py:149, core.py:118-129
    s2 = comm.all_gather_vec(np.einsum("ij,ij->j", W_local, W_local), device)
    tot = np.sum(s2, axis=0)
    Z_local = np.where(tot[None, :] > 0, W_local / np.sqrt(np.where(tot > 0, tot, 1.0))[None, :], 0.0)
    Z = np.column_stack([_gather_ragged(comm, np.ascontiguousarray(Z_local[:, j]), offset, n_global, device)
                         for j in range(m)])
    loadings = SparseLoadings(Z)
    return loadings, RunReport(history, len(history) - 1, time.perf_counter() - start,
                               loadings.nnz_per_component(), converged, [history])

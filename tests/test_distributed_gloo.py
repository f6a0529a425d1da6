"""World-size-2 gloo tests of the column-sharded solve driver (CPU only).

The device shard loop is replaced by a test-side loop that restates the
device semantics (sweep -> exchange vector [g | f | nnz | sum w^2 | 0] ->
step) on the rank's NumPy shard; everything else -- partitioning, the
global max-norm start with lowest-global-index ties, the activation-limit
max, the per-iteration all-reduce, the ||w||^2 all-reduce and the loadings
gather -- is the product code in paper_1312_6182_b200/distributed.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

WORLD = 2


class OracleShardLoop:
    def __init__(self, A_local, penalty, gamma, tol, max_iter):
        self.A = A_local.values
        self.penalty, self.gamma, self.tol, self.max_iter = penalty, gamma, tol, max_iter
        self.buf = torch.zeros(self.A.shape[0] + 4, dtype=torch.float64)

    def start(self, x0):
        self.x = np.array(x0, dtype=np.float64)
        self.k, self.done, self.conv, self.f_prev, self.hist = 0, False, False, 0.0, []
        self.w = np.zeros(self.A.shape[1])

    def enqueue_sweep(self):
        if self.done:
            return
        c = self.A.T @ self.x
        self.w = oracle.threshold(c, self.gamma, self.penalty)
        g = self.A @ self.w
        vec = np.concatenate([g, [oracle.su_objective(c, self.gamma, self.penalty),
                                  np.count_nonzero(self.w), self.w @ self.w, 0.0]])
        self.buf.copy_(torch.from_numpy(vec))

    def exchange(self):
        return self.buf

    def enqueue_step(self):
        if self.done:
            return
        v = self.buf.numpy()
        p = self.A.shape[0]
        f = float(v[p])
        self.hist.append(f)
        if self.k >= 1 and abs(f - self.f_prev) < self.tol * max(abs(self.f_prev), 1e-30):
            self.done, self.conv = True, True
            return
        if self.k >= self.max_iter:
            self.done = True
            return
        g = v[:p]
        nrm = np.linalg.norm(g)
        if nrm == 0.0:
            self.done, self.conv = True, True
            return
        self.x = g / nrm
        self.f_prev = f
        self.k += 1

    def poll(self):
        return self.done, self.k, self.conv

    def result(self):
        return self.x, list(self.hist), self.conv, self.w


class HostShard:
    """Stand-in for a DataMatrix shard: .values/.norms/.column/.p/.n."""

    def __init__(self, values):
        self.values = np.asfortranarray(values)
        self.p, self.n = values.shape
        self.norms = np.linalg.norm(self.values, axis=0)

    def column(self, i):
        return self.values[:, i].copy()


class OracleBlockShardLoop:
    """Test-side restatement of the device block loop semantics on a shard."""

    def __init__(self, A_local, penalty, m, gamma, mu, tol, max_iter):
        self.A = A_local.values
        self.penalty, self.m, self.tol, self.max_iter = penalty, m, tol, max_iter
        self.gamma = np.broadcast_to(np.asarray(gamma, float), (m,)).copy()
        self.mu = np.broadcast_to(np.asarray(mu, float), (m,)).copy()
        self.buf = torch.zeros(self.A.shape[0] * m + 2, dtype=torch.float64)

    def start(self, M, orthonormalize):
        if orthonormalize:
            Q, R = np.linalg.qr(M)
            self.X = Q * np.sign(np.diagonal(R))
        else:
            self.X = np.array(M)
        self.k, self.done, self.conv, self.f_prev, self.hist = 0, False, False, 0.0, []
        self.rank_fail, self.rank = False, 0
        self.W = np.zeros((self.A.shape[1], self.m))

    def enqueue_sweep(self):
        if self.done:
            return
        C = self.A.T @ self.X
        self.W = np.column_stack([oracle.threshold(self.mu[j] * C[:, j], self.gamma[j], self.penalty)
                                  for j in range(self.m)])
        f = oracle.block_objective(C, self.gamma, self.mu, self.penalty)
        G = self.A @ self.W
        self.buf.copy_(torch.from_numpy(np.concatenate([G.ravel(order="F"), [f, 0.0]])))

    def exchange(self):
        return self.buf

    def enqueue_step(self):
        if self.done:
            return
        v = self.buf.numpy()
        p = self.A.shape[0]
        f = float(v[p * self.m])
        self.hist.append(f)
        if self.k >= 1 and abs(f - self.f_prev) < self.tol * max(abs(self.f_prev), 1e-30):
            self.done, self.conv = True, True
            return
        if self.k >= self.max_iter:
            self.done = True
            return
        G = v[: p * self.m].reshape((p, self.m), order="F") * (2.0 * self.mu)[None, :]
        try:
            self.X = oracle.polar(G)
        except oracle.OracleRankDeficiency as err:
            self.done, self.rank_fail, self.rank = True, True, err.rank
            return
        self.f_prev = f
        self.k += 1

    def poll(self):
        return self.done, self.k, self.conv

    def result(self):
        return self.X, list(self.hist), self.conv, self.W, self.rank_fail, self.rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_1312_6182_b200 import SolverConfig
        from paper_1312_6182_b200.distributed import Comm, column_partition, solve_single_unit_sharded

        A = case["A"]
        off, cnt = column_partition(A.shape[1], WORLD)[rank]
        shard = HostShard(A[:, off:off + cnt])
        cfg = SolverConfig(penalty=case["penalty"], gamma=case["gamma"], **case.get("cfg", {}))
        loadings, report = solve_single_unit_sharded(shard, cfg, off, A.shape[1], comm=Comm(),
                                                     loop_factory=OracleShardLoop, poll_every=3)
        out[rank] = (loadings.values[:, 0].copy(), list(report.objective_history), report.converged)
    finally:
        dist.destroy_process_group()


def _run(case):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), case, out), nprocs=WORLD, join=True)
    return dict(out)


CASES = {
    "sl1_gauss": dict(seed=0, shape=(60, 301), penalty="l1", rule=lambda nm: 0.1 * nm),
    "sl0_gauss": dict(seed=1, shape=(40, 500), penalty="l0", rule=lambda nm: (0.15 * nm) ** 2),
    "sl1_random_init": dict(seed=2, shape=(30, 201), penalty="l1", rule=lambda nm: 0.2 * nm,
                            cfg=dict(init="random_orthonormal", seed=5)),
    "inactive": dict(seed=3, shape=(10, 20), penalty="l1", rule=lambda nm: 2.0 * nm),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_sharded_solve_matches_oracle(name):
    spec = CASES[name]
    A = np.random.default_rng(spec["seed"]).standard_normal(spec["shape"])
    gamma = float(spec["rule"](np.linalg.norm(A, axis=0).max()))
    case = {"A": A, "penalty": spec["penalty"], "gamma": gamma, "cfg": spec.get("cfg", {})}
    res = _run(case)
    cfg = spec.get("cfg", {})
    z_ref, hist_ref, conv_ref, _ = oracle.su_solve(A, gamma, spec["penalty"], **cfg)
    for rank in range(WORLD):
        z, hist, conv = res[rank]
        assert conv == conv_ref
        assert len(hist) == len(hist_ref)
        np.testing.assert_allclose(hist, hist_ref, rtol=1e-12, atol=1e-14)
        assert np.array_equal(z != 0, z_ref != 0)
        np.testing.assert_allclose(z, z_ref, rtol=1e-10, atol=1e-12)
    np.testing.assert_array_equal(res[0][0], res[1][0])


def _tie_worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_1312_6182_b200.distributed import Comm, global_max_norm_start

        p = 3
        # both shards hold an equal max-norm column; rank 0's is the lower global index
        cols = {0: np.array([[0.0, 3.0], [0.0, 4.0], [1.0, 0.0]]), 1: np.array([[5.0, 1.0], [0.0, 0.0], [0.0, 0.0]])}
        local = cols[rank]
        norms = np.linalg.norm(local, axis=0)
        x0, val = global_max_norm_start(norms, rank * 2, lambda i: local[:, i].copy(), Comm(), p)
        out[rank] = (x0.copy(), val)
    finally:
        dist.destroy_process_group()


def test_global_max_norm_tie_breaks_to_lowest_index():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_tie_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    for rank in range(WORLD):
        x0, val = out[rank]
        assert val == 5.0
        np.testing.assert_allclose(x0, [0.6, 0.8, 0.0])  # global column 1 (rank 0), not column 2


def _block_worker(rank, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_1312_6182_b200 import RankDeficiencyError, SolverConfig
        from paper_1312_6182_b200.distributed import Comm, column_partition, solve_block_sharded

        A = case["A"]
        off, cnt = column_partition(A.shape[1], WORLD)[rank]
        shard = HostShard(A[:, off:off + cnt])
        cfg = SolverConfig(penalty=case["penalty"], mode="block", m=case["m"], gamma=case["gamma"],
                           mu=case["mu"], **case.get("cfg", {}))
        try:
            loadings, report = solve_block_sharded(shard, cfg, off, A.shape[1], comm=Comm(),
                                                   loop_factory=OracleBlockShardLoop, poll_every=3)
            out[rank] = ("ok", loadings.values.copy(), list(report.objective_history), report.converged)
        except RankDeficiencyError as err:
            out[rank] = ("rank", err.rank, err.iteration, list(err.history))
    finally:
        dist.destroy_process_group()


BLOCK_CASES = {
    "bl1_maxnorm": dict(seed=4, shape=(30, 201), penalty="l1", m=3, mu=1.0, rule=lambda nm: 0.1 * nm),
    "bl0_mu_random": dict(seed=5, shape=(25, 150), penalty="l0", m=4, mu=[1.0, 0.9, 0.8, 0.7],
                          rule=lambda nm: (0.12 * nm) ** 2, cfg=dict(init="random_orthonormal", seed=2)),
}


@pytest.mark.parametrize("name", sorted(BLOCK_CASES))
def test_sharded_block_solve_matches_oracle(name):
    spec = BLOCK_CASES[name]
    A = np.random.default_rng(spec["seed"]).standard_normal(spec["shape"])
    gamma = float(spec["rule"](np.linalg.norm(A, axis=0).max()))
    case = {"A": A, "penalty": spec["penalty"], "gamma": gamma, "m": spec["m"], "mu": spec["mu"],
            "cfg": spec.get("cfg", {})}
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_block_worker, args=(_free_port(), case, out), nprocs=WORLD, join=True)
    cfg = dict(spec.get("cfg", {}))
    init = cfg.pop("init", "max_norm_column")
    Z_ref, hist_ref, conv_ref, _ = oracle.block_solve(A, spec["m"], gamma, spec["mu"], spec["penalty"],
                                                      init=init, **cfg)
    for rank in range(WORLD):
        status, Z, hist, conv = out[rank]
        assert status == "ok"
        assert conv == conv_ref and len(hist) == len(hist_ref)
        np.testing.assert_allclose(hist, hist_ref, rtol=1e-12, atol=1e-14)
        assert np.array_equal(Z != 0, Z_ref != 0)
        np.testing.assert_allclose(Z, Z_ref, rtol=1e-9, atol=1e-12)


def _px_decision_worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import torch

        from paper_1312_6182_b200.distributed import Comm, peer_exchange_available

        comm = Comm()
        # CPU ranks, and ranks sharing one GPU index, never take the peer-memory path
        # (spinning ranks on one device could wait on each other); all ranks agree
        out[rank] = (peer_exchange_available(comm, "cpu"),
                     peer_exchange_available(comm, torch.device("cpu")))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_decision_on_cpu_ranks():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_px_decision_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    assert all(out[r] == (False, False) for r in range(WORLD))


class _FakePeerExchange:
    """Stand-in for PeerExchange: sums through gloo (correct), adds a bias
    on one rank (a broken peer path), or raises (a peer path that cannot
    run) -- exercising px_self_test's agreement logic without a GPU."""

    def __init__(self, mode, comm):
        self.mode, self.comm = mode, comm
        # "broken": rank 1 could not open its peers' buffers (PeerExchange.ok)
        self.ok = not (mode == "broken" and comm.rank == 1)

    def all_reduce(self, t):
        assert self.ok, "a rank whose construction failed must not launch the exchange"
        self.comm.all_reduce_sum(t)  # the exchange itself (a device kernel in the real class)
        if self.mode == "raise" and self.comm.rank == 1:
            raise RuntimeError("peer exchange timed out")  # e.g. this rank's bounded wait expired
        if self.mode == "wrong" and self.comm.rank == 0:
            t += 1e-6


def _self_test_worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_1312_6182_b200.distributed as d

        comm = d.Comm()
        # px_self_test synchronises the device; on CPU ranks make that a no-op
        torch.cuda.synchronize = lambda *a, **k: None
        res = {}
        for mode in ("ok", "wrong", "raise", "broken"):
            res[mode] = d.px_self_test(_FakePeerExchange(mode, comm), comm, torch.device("cpu"), 300)
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_peer_exchange_self_test_agreement():
    """Every rank keeps the peer path only when all ranks reproduced the
    torch.distributed sum; one wrong or failing rank, or one that could not
    open its peers' buffers, sends all to NCCL (and none of them launches)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_self_test_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    for r in range(WORLD):
        assert out[r] == {"ok": True, "wrong": False, "raise": False, "broken": False}, out[r]

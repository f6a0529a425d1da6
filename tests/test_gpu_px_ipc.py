"""The peer-memory exchange across real processes (csrc/px_kernels.cuh,
gps_px_*): `world` processes on cuda:0, each with its own CUDA context,
export their symmetric buffers with cudaIpcGetMemHandle, all-gather the
handles over gloo and open every peer's with cudaIpcOpenMemHandle -- the
path a multi-GPU job takes (distributed.PeerExchange), minus NVLink.

One GPU cannot run ranks whose kernels wait on each other (separate
contexts are time-sliced), so every exchange runs as its two halves
(gps_px_allreduce_phase / gps_px_reduce_phase): every rank pushes its vector
into every rank's IPC-mapped slots and release-stores its epoch flags
(phase 1), a host barrier, then every rank acquires the flags -- already set
-- and sums the slots in rank order (phase 2).  Several rounds cover both
slot parities and the epoch protocol; the result must be bitwise the
rank-order sum on every rank.  A rank that skips its push leaves its peers
to time out (error flag) rather than hang."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, json
import numpy as np
sys.path.insert(0, %(root)r)
sys.path.insert(0, os.path.join(%(root)r, "tests"))
import torch, torch.distributed as dist
from paper_1312_6182_b200 import _native
from test_gpu_peer_exchange import k2_reference, rank_order_sum
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
torch.cuda.set_device(0)
L = _native.lib()
ctx = _native.context(0)
out = {"rank": rank, "checks": []}

def open_px(count):
    h = _native._vp()
    _native.check(L.gps_px_create(ctx.handle, world, rank, count, _native.C.byref(h)))
    size = L.gps_px_handle_size()
    mine = (_native.C.c_char * size)()
    _native.check(L.gps_px_ipc_handle(h, mine))
    handles = [None] * world
    dist.all_gather_object(handles, bytes(mine))
    for peer, hb in enumerate(handles):
        _native.check(L.gps_px_open(h, peer, (_native.C.c_char * size).from_buffer_copy(hb)))
    return h

def phases(launch):
    # push, host barrier, gather: no kernel of one process waits on another's
    launch(1); ctx.sync(); dist.barrier()
    launch(2); ctx.sync(); dist.barrier()

def err_flag(h):
    e = _native.C.c_int(-1)
    _native.check(L.gps_px_error(h, _native.C.byref(e)))
    return e.value

# 1. standalone all-reduce, 4 rounds (epochs 1..4, both parities)
for count in (5, 4100, 3 * 4096 + 7):
    h = open_px(count)
    vecs = [np.random.default_rng(100 * q + count).standard_normal(count) * 10.0 ** q for q in range(world)]
    for k in range(4):
        t = torch.tensor(vecs[rank] * (k + 1), device="cuda:0")
        torch.cuda.synchronize()
        phases(lambda ph: _native.check(L.gps_px_allreduce_phase(h, _native._vp(t.data_ptr()), ph)))
        ref = rank_order_sum([v * (k + 1) for v in vecs])
        out["checks"].append(["allreduce", count, k, bool(np.array_equal(t.cpu().numpy(), ref))])
    out["checks"].append(["allreduce_err", count, 0, err_flag(h) == 0])
    L.gps_px_destroy(h)

# 2. the fused K2 reduction + exchange (su_reduce_px_kernel) on CTA partials
for rows, nparts, nparts_s in ((4096, 148, 148), (3 * 4096 + 96, 32, 5)):
    h = open_px(rows + 4)
    pg = [np.random.default_rng(7 * q + rows).standard_normal((nparts, rows)) for q in range(world)]
    ps = [np.random.default_rng(9 * q + rows).standard_normal((nparts_s, 4)) for q in range(world)]
    for k in range(3):
        dg = torch.tensor(pg[rank] * (k + 1), device="cuda:0")
        ds = torch.tensor(ps[rank] * (k + 1), device="cuda:0")
        ex = torch.zeros(rows + 4, dtype=torch.float64, device="cuda:0")
        torch.cuda.synchronize()
        phases(lambda ph: _native.check(L.gps_px_reduce_phase(h, _native._vp(dg.data_ptr()), _native._vp(ds.data_ptr()),
                                                              nparts, rows, nparts_s, _native._vp(ex.data_ptr()), ph)))
        ref = rank_order_sum([k2_reference(pg[q] * (k + 1), ps[q] * (k + 1), rows) for q in range(world)])
        out["checks"].append(["reduce", rows, k, bool(np.array_equal(ex.cpu().numpy(), ref))])
    out["checks"].append(["reduce_err", rows, 0, err_flag(h) == 0])
    L.gps_px_destroy(h)

# 3. the last rank skips its push: every other rank's gather times out
h = open_px(4100)
_native.check(L.gps_px_set_timeout(h, 0.5))
t = torch.ones(4100, dtype=torch.float64, device="cuda:0")
torch.cuda.synchronize()
if rank != world - 1:
    _native.check(L.gps_px_allreduce_phase(h, _native._vp(t.data_ptr()), 1))
ctx.sync(); dist.barrier()
if rank != world - 1:
    _native.check(L.gps_px_allreduce_phase(h, _native._vp(t.data_ptr()), 2))
    ctx.sync()
    out["checks"].append(["timeout", 4100, 0, err_flag(h) == 1 and bool(torch.all(t == 1).item())])
dist.barrier()
L.gps_px_destroy(h)
print("RESULT" + json.dumps(out), flush=True)
dist.destroy_process_group()
"""


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_ipc_exchange_across_processes(world):
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   LOCAL_RANK="0", GPSPCA_PX_TIMEOUT_S="20")
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER % {"root": ROOT}], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        try:
            so, se = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        assert p.returncode == 0, se[-3000:]
        outs.append(so)
    for so in outs:
        line = [ln for ln in so.splitlines() if ln.startswith("RESULT")]
        assert line, so[-2000:]
        res = json.loads(line[0][len("RESULT"):])
        bad = [c for c in res["checks"] if not c[3]]
        assert not bad, (res["rank"], bad)
        n_timeout = 0 if res["rank"] == world - 1 else 1
        assert len(res["checks"]) == 3 * 5 + 2 * 4 + n_timeout

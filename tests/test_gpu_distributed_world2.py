"""The sharded device drivers at world size 2 on one GPU: two processes,
each owning a column shard as its own DataMatrix on cuda:0, exchanging
through a gloo process group (the collective is host-mediated, so the two
ranks' kernels never wait on each other).  Checks the sharded device path --
shard-local sweeps, the all-reduced exchange vector, the identical step on
every rank, the global start column and the gathered loadings -- against the
unsharded device solve and the fp64 oracle."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, json
import numpy as np
sys.path.insert(0, %(root)r)
import torch, torch.distributed as dist
import paper_1312_6182_b200 as gps
from paper_1312_6182_b200.distributed import column_partition, solve_single_unit_sharded, solve_block_sharded
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
torch.cuda.set_device(0)
rng = np.random.default_rng(17)
A = rng.standard_normal((300, 5001)).astype(np.float32)      # ragged split
B = rng.standard_normal((200, 3001))                           # fp64, block
out = {}
for name, M, cfg in (
        ("su_l1", A, gps.SolverConfig(penalty="l1", gamma=0.1 * float(np.linalg.norm(A.astype(np.float64), axis=0).max()))),
        ("su_l0", A, gps.SolverConfig(penalty="l0", gamma=(0.1 * float(np.linalg.norm(A.astype(np.float64), axis=0).max())) ** 2)),
        ("bl1", B, gps.SolverConfig(penalty="l1", mode="block", m=5, gamma=0.1 * float(np.linalg.norm(B, axis=0).max()))),
        ("bl0_tc", A, gps.SolverConfig(penalty="l0", mode="block", m=8, gamma=(0.05 * float(np.linalg.norm(A.astype(np.float64), axis=0).max())) ** 2))):
    off, nl = column_partition(M.shape[1], world)[rank]
    local = gps.DataMatrix(np.ascontiguousarray(M[:, off:off + nl]))
    solve = solve_single_unit_sharded if cfg.mode == "single_unit" else solve_block_sharded
    z, r = solve(local, cfg, off, M.shape[1], device=torch.device("cuda", 0))
    out[name] = {"iters": r.iterations, "hist": list(r.objective_history), "z": z.values.tolist()}
if rank == 0:
    print("RESULT" + json.dumps(out))
dist.destroy_process_group()
"""


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_solves_world2_on_one_gpu():
    import json

    import paper_1312_6182_b200 as gps

    port = _port()
    procs = []
    for rank in range(2):
        env = {**os.environ, "RANK": str(rank), "WORLD_SIZE": "2", "LOCAL_RANK": "0", "GPSPCA_DEVICE": "0",
               "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)}
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER % {"root": ROOT}], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    res = json.loads(next(l for l in outs[0][0].splitlines() if l.startswith("RESULT"))[6:])

    rng = np.random.default_rng(17)
    A = rng.standard_normal((300, 5001)).astype(np.float32)
    B = rng.standard_normal((200, 3001))
    gA = 0.1 * float(np.linalg.norm(A.astype(np.float64), axis=0).max())
    gB = 0.1 * float(np.linalg.norm(B, axis=0).max())
    refs = {
        "su_l1": gps.solve_single_unit(A, gps.SolverConfig(penalty="l1", gamma=gA)),
        "su_l0": gps.solve_single_unit(A, gps.SolverConfig(penalty="l0", gamma=gA * gA)),
        "bl1": gps.solve_block(B, gps.SolverConfig(penalty="l1", mode="block", m=5, gamma=gB)),
        "bl0_tc": gps.solve_block(A, gps.SolverConfig(penalty="l0", mode="block", m=8, gamma=(0.5 * gA) ** 2)),
    }
    for name, (z_ref, r_ref) in refs.items():
        got = res[name]
        # the shard boundary changes only the order of the fixed-order sums
        assert got["iters"] == r_ref.iterations, name
        np.testing.assert_allclose(got["hist"], r_ref.objective_history, rtol=1e-9, err_msg=name)
        np.testing.assert_allclose(np.asarray(got["z"]), z_ref.values, atol=1e-7, err_msg=name)

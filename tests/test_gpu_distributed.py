"""The sharded drivers on a real device: world-size-1 NCCL process group,
torch-owned exchange buffers all-reduced in place on the engine's stream.
(Multi-rank host logic is covered by tests/test_distributed_gloo.py.)"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

gps = pytest.importorskip("paper_1312_6182_b200")
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_sharded_single_unit_world1(nccl_group):
    from paper_1312_6182_b200.distributed import solve_single_unit_sharded

    rng = np.random.default_rng(3)
    A32 = rng.standard_normal((300, 4000)).astype(np.float32)
    A = gps.DataMatrix(A32)
    cfg = gps.SolverConfig(penalty="l1", gamma=0.1 * float(A.norms.max()))
    z_ref, r_ref = gps.solve_single_unit(A, cfg)
    z, r = solve_single_unit_sharded(A, cfg, 0, A.n, device=torch.device("cuda", 0))
    assert r.iterations == r_ref.iterations
    np.testing.assert_allclose(r.objective_history, r_ref.objective_history, rtol=1e-12)
    np.testing.assert_allclose(z.values, z_ref.values, rtol=1e-10, atol=1e-14)


def test_sharded_block_world1(nccl_group):
    from paper_1312_6182_b200.distributed import solve_block_sharded

    rng = np.random.default_rng(4)
    A = gps.DataMatrix(rng.standard_normal((200, 3000)))
    cfg = gps.SolverConfig(penalty="l1", mode="block", m=5, gamma=0.1 * float(A.norms.max()))
    z_ref, r_ref = gps.solve_block(A, cfg)
    z, r = solve_block_sharded(A, cfg, 0, A.n, device=torch.device("cuda", 0))
    assert r.iterations == r_ref.iterations
    np.testing.assert_allclose(r.objective_history, r_ref.objective_history, rtol=1e-12)
    np.testing.assert_allclose(z.values, z_ref.values, rtol=1e-9, atol=1e-12)

"""Two C4-shaped block iterations (BL0 m=64, p=8192, n=2^21 fp32) on the tensor-core path, for ncu."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1312_6182_b200 as gps
    from paper_1312_6182_b200 import _native
    from paper_1312_6182_b200.block import BlockLoop, _top_m_columns

    p, n, m = 8192, int(os.environ.get("TC_N", 1 << 21)), 64
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    At = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float32)
    A = gps.DataMatrix.from_device(At.data_ptr(), p, n, owner=At)
    gamma = np.full(m, (0.1 * float(A.norms.max())) ** 2)
    loop = BlockLoop(A, "l0", m, gamma, np.linspace(1, 0.5, m), 0.0, 10)
    loop.start_columns(_top_m_columns(np.asarray(A.norms), m))
    L = _native.lib()
    for it in range(int(os.environ.get("TC_ITERS", 2))):
        A.context.sync()
        t0 = time.perf_counter()
        _native.check(L.gps_bk_enqueue_sweep(loop.handle))
        _native.check(L.gps_bk_enqueue_step(loop.handle))
        A.context.sync()
        print(f"iteration {it}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)


if __name__ == "__main__":
    main()

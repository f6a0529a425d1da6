"""One C3-shaped block iteration (BL1 m=10, p=4096, n=2^21 fp32) for ncu."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1312_6182_b200 as gps
    from paper_1312_6182_b200 import _native
    from paper_1312_6182_b200.block import BlockLoop, _top_m_columns

    p, n, m = 4096, 1 << 21, 10
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    At = torch.randn((n, p), generator=g, device="cuda", dtype=torch.float32)
    A = gps.DataMatrix.from_device(At.data_ptr(), p, n, owner=At)
    gamma = np.full(m, 0.1 * float(A.norms.max()))
    loop = BlockLoop(A, "l1", m, gamma, np.ones(m), 0.0, 10)
    loop.start_columns(_top_m_columns(np.asarray(A.norms), m))
    L = _native.lib()
    for _ in range(2):
        _native.check(L.gps_bk_enqueue_sweep(loop.handle))
        _native.check(L.gps_bk_enqueue_step(loop.handle))
    A.context.sync()
    print("ok")


if __name__ == "__main__":
    main()

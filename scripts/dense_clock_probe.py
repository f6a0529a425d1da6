"""bench.su_dense_line three times with clocks (is the dense sweep power-capped?)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1312_6182_b200 as gps  # noqa: E402
from paper_1312_6182_b200 import _native  # noqa: E402

p, n = 4096, 1 << 20
dev = torch.device("cuda", 0)
At = bench.make_c2(torch, p, n, 0, n, dev)
torch.cuda.synchronize()
A = gps.DataMatrix.from_device(At.data_ptr(), p, n, ld=p, dtype=np.float32, device=0)
ctx = _native.context(0)
for rep in range(4):
    r = bench.su_dense_line(torch, gps, ctx, dev, A, p, n)
    print(rep, f"{r['ms_per_iter']:.3f} ms", r["clocks"], flush=True)
    time.sleep(3)

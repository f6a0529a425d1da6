"""K1 at C2 size with gamma = 0 (every column active): a few device-resident
iterations for ncu (`-k regex:su_sweep -c 1 --set full`) and a CUDA-event
timing.  Usage: python scripts/su_dense_probe.py [gamma_frac] [iters]."""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1312_6182_b200 as gps  # noqa: E402
from paper_1312_6182_b200 import _native  # noqa: E402

frac = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p, n = 4096, 1 << 20
dev = torch.device("cuda", 0)
At = bench.make_c2(torch, p, n, 0, n, dev)
if os.environ.get("PROBE_COPY"):  # engine-owned copy, as bench.py's C2 matrix
    A = gps.DataMatrix.from_device(At.data_ptr(), p, n, ld=p, dtype=np.float32, device=0)
else:
    A = gps.DataMatrix.from_device(At.data_ptr(), p, n, owner=At, device=0)
gamma = (frac * float(A.norms.max())) ** 2
i = int(np.argmax(A.norms))
loop = gps.single_unit.PowerLoop(A, "l0", gamma, 0.0, iters + 4)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
_native.context().set_stream(stream.cuda_stream)
loop.start(A.column(i) / A.norms[i])
L = _native.lib()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
_native.check(L.gps_su_enqueue(loop.handle, 7))
e0.record(stream)
for _ in range(iters):
    _native.check(L.gps_su_enqueue(loop.handle, 7))
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
print(f"gamma_frac={frac} ms/iter={ms:.3f} GB/s={p * n * 4 / ms / 1e6:.0f}")

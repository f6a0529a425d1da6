"""Block iteration time at the C3 shape (p=4096, n=2^21 fp32) for several m,
CUDA-core sweep (GPSPCA_NO_TC=1) vs tensor-core sweep (GPSPCA_TC_MIN_M=1)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys, time
import numpy as np
sys.path.insert(0, %r)
import torch
import paper_1312_6182_b200 as gps
from paper_1312_6182_b200 import _native
from paper_1312_6182_b200.block import BlockLoop, _top_m_columns
p, n, m = 4096, int(os.environ.get('TC_N', 1 << 21)), int(os.environ['TC_M'])
g = torch.Generator(device='cuda'); g.manual_seed(3)
At = torch.randn((n, p), generator=g, device='cuda', dtype=torch.float32)
A = gps.DataMatrix.from_device(At.data_ptr(), p, n, owner=At)
top = float(A.norms.max())
loop = BlockLoop(A, 'l1', m, np.full(m, 0.1 * top), np.ones(m), 0.0, 20)
loop.start_columns(_top_m_columns(np.asarray(A.norms), m))
L = _native.lib()
ts = []
for it in range(6):
    A.context.sync(); t0 = time.perf_counter()
    _native.check(L.gps_bk_enqueue_sweep(loop.handle)); _native.check(L.gps_bk_enqueue_step(loop.handle))
    A.context.sync(); ts.append(time.perf_counter() - t0)
t = min(ts[2:])
print(f"m={m:3d} {os.environ.get('MODE'):4s}: {t*1e3:7.3f} ms/iter  {1/t:7.1f} it/s  A-stream(1 read) {p*n*4/t/1e9:6.0f} GB/s", flush=True)
""" % ROOT

for m in (4, 5, 8, 10, 16, 32):
    for mode in ("cc", "tc"):
        env = {**os.environ, "TC_M": str(m), "MODE": mode}
        env.update({"GPSPCA_NO_TC": "1"} if mode == "cc" else {"GPSPCA_TC_MIN_M": "1"})
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        print(r.stdout.strip() or r.stderr[-600:], flush=True)

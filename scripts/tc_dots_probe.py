"""Time the tensor-core block sweep (tc_split_x + tc_dots + tc_refine +
tc_update + reduce) at the C4 shape (TC_P / TC_N / TC_M override it) under
GPSPCA_TC_PROBE variants (timing experiments only)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r"""
import os, sys, time
import numpy as np
sys.path.insert(0, %r)
import torch
import paper_1312_6182_b200 as gps
from paper_1312_6182_b200 import _native
from paper_1312_6182_b200.block import BlockLoop, _top_m_columns
p, n, m = int(os.environ.get('TC_P', 8192)), int(os.environ.get('TC_N', 1 << 20)), int(os.environ.get('TC_M', 64))
g = torch.Generator(device='cuda'); g.manual_seed(4)
At = torch.randn((n, p), generator=g, device='cuda', dtype=torch.float32)
A = gps.DataMatrix.from_device(At.data_ptr(), p, n, owner=At)
gamma = np.full(m, (0.1 * float(A.norms.max())) ** 2)
loop = BlockLoop(A, 'l0', m, gamma, np.linspace(1, 0.5, m), 0.0, 10)
loop.start_columns(_top_m_columns(np.asarray(A.norms), m))
L = _native.lib()
ts = []
for it in range(6):
    A.context.sync(); t0 = time.perf_counter()
    _native.check(L.gps_bk_enqueue_sweep(loop.handle))
    A.context.sync(); ts.append(time.perf_counter() - t0)
t = min(ts[2:])
if int(os.environ.get('GPSPCA_TC_PROBE', '0')) & 64:
    import ctypes as C
    fn = L.gpsdbg_tc_profile
    fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int, C.c_int]
    fn(None, 0, 1)
    _native.check(L.gps_bk_enqueue_sweep(loop.handle)); A.context.sync()
    buf = (C.c_ulonglong * 16)()
    fn(buf, 16, 0)
    v = list(buf)
    chunks = (n // 128) * ((p + 63) // 64)
    names = {1: 'A prod wait a_empty', 2: 'X prod wait x_empty', 3: 'MMA wait tempty', 4: 'MMA wait lo_full',
             5: 'MMA wait x_full', 6: 'MMA role total', 7: 'conv wait a_full', 8: 'conv wait lo_empty',
             9: 'conv tmem st', 10: 'conv role total', 11: 'epi wait tfull', 12: 'epi drain', 13: 'epi role total'}
    for k, nm in names.items():
        print(f"  {nm:22s} {v[k] / chunks:8.1f} clk/chunk")
print(f"probe={os.environ.get('GPSPCA_TC_PROBE','0'):>3} p={p} n={n} m={m}: sweep {t*1e3:.3f} ms  A-stream {p*n*4/t/1e9:.0f} GB/s")
""" % ROOT

if os.environ.get("TC_INLINE"):
    exec(CHILD)
    sys.exit(0)
for probe in sys.argv[1:] or ["0", "16", "17", "18", "20", "24", "31"]:
    env = {**os.environ, "GPSPCA_TC_PROBE": probe}
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    print(r.stdout.strip() or r.stderr[-800:], flush=True)

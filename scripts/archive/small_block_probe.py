"""A small block solve (the paper grid's P = 1000, N = 10000, m = 5) for an
ncu launch list: per-kernel fixed costs of the block iteration."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_6182_b200 as gps  # noqa: E402

dt = np.float64 if os.environ.get("SB_DTYPE", "f64") == "f64" else np.float32
A = np.random.default_rng(0).standard_normal((1000, 10000)).astype(dt)
D = gps.DataMatrix(A, dtype=dt)
g = 0.05 * float(np.linalg.norm(A.astype(np.float64), axis=0).max())
cfg = gps.SolverConfig(penalty="l1", mode="block", m=5, gamma=g, max_iter=int(os.environ.get("SB_ITERS", 40)), tol=1e-15)
gps.solve_block(D, cfg)
t0 = time.perf_counter()
_, r = gps.solve_block(D, cfg)
t = time.perf_counter() - t0
print(f"{np.dtype(dt).name}: {r.iterations} iterations, {t / r.iterations * 1e6:.1f} us/iteration, "
      f"{r.kernel_launches} launches")

# phase split of one solve (host wall clock)
from paper_1312_6182_b200.block import BlockLoop, _top_m_columns  # noqa: E402

for rep in range(2):
    t = [time.perf_counter()]
    loop = BlockLoop(D, "l1", 5, np.full(5, g), np.ones(5), 1e-15, cfg.max_iter)
    t.append(time.perf_counter())
    loop.start_columns(_top_m_columns(np.asarray(D.norms), 5))
    t.append(time.perf_counter())
    X, hist, conv, W = loop.run(8)
    t.append(time.perf_counter())
    del loop
    t.append(time.perf_counter())
    print("create %.0f us, start %.0f us, run %.0f us (%d its), destroy %.0f us" % (
        (t[1] - t[0]) * 1e6, (t[2] - t[1]) * 1e6, (t[3] - t[2]) * 1e6, len(hist) - 1, (t[4] - t[3]) * 1e6))

"""Smoke-check the tensor-core block sweep (m >= 16) against the fp64 oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1312_6182_b200 as gps  # noqa: E402


def check(p, n, m, pen, seed=0):
    rng = np.random.default_rng(seed)
    A32 = rng.standard_normal((p, n)).astype(np.float32)
    A = gps.DataMatrix(np.asfortranarray(A32))
    Q, _ = np.linalg.qr(rng.standard_normal((p, m)))
    gamma = np.full(m, 2.0 if pen == "l1" else 4.0)
    mu = np.linspace(1.0, 0.6, m)
    A64 = A32.astype(np.float64)
    C = A64.T @ Q
    f_ref = oracle.block_objective(C, gamma, mu, pen)
    G_ref = oracle.block_gradient(A64, C, gamma, mu, pen)
    f = (gps.objective_bl1 if pen == "l1" else gps.objective_bl0)(A, Q, gamma, mu)
    G = gps.ascent_direction_block(A, Q, gamma, mu, pen)
    relG = np.abs(G - G_ref).max() / np.abs(G_ref).max()
    print(f"p={p} n={n} m={m} {pen}: f={f:.8e} ref={f_ref:.8e} rel={abs(f-f_ref)/abs(f_ref):.2e} G rel={relG:.2e}",
          flush=True)
    return abs(f - f_ref) / abs(f_ref) < 1e-4 and relG < 1e-4


ok = True
for args in [(256, 1000, 16, "l1"), (256, 1000, 16, "l0"), (512, 3000, 32, "l1"), (4096, 20000, 64, "l0"),
             (8192, 16384, 64, "l1")]:
    ok &= check(*args)
print("TC PROBE", "OK" if ok else "FAIL")

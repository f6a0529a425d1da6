"""One timing-harness solve (bl0, N=10000, P=1000, m=5, gamma=0.01) per instance, for ncu."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1312_6182_b200.timing import fit_projection  # noqa: E402

for inst in [int(a) for a in sys.argv[1:]] or [0, 1, 2]:
    rng = np.random.default_rng([0, 10000, inst])
    A = rng.standard_normal((1000, 10000))
    t = time.perf_counter()
    Z, mean, rep = fit_projection(A, os.environ.get("VARIANT", "bl0"), 5, 0.01, seed=[0, 10000, inst], center=False)
    dt = time.perf_counter() - t
    print(inst, f"{dt * 1e3:.1f} ms", rep.iterations, f"{dt / rep.iterations * 1e6:.1f} us/it", flush=True)

import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1312_6182_b200.timing import fit_projection
import paper_1312_6182_b200 as gps
for rep in range(3):
    for inst in range(3):
        rng = np.random.default_rng([0, 1000, inst])
        A = rng.standard_normal((100, 1000))
        t = time.perf_counter()
        Z, mean, rep_ = fit_projection(A, "bl0", 5, 0.01, seed=[0, 1000, inst], center=False)
        dt = time.perf_counter() - t
        print(rep, inst, f"{dt*1e3:.1f} ms", rep_.iterations, f"{dt/rep_.iterations*1e6:.1f} us/it")

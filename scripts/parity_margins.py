"""Largest deviation of the device solves from the reference's golden outputs
(tests/golden/solves.json), per case and storage dtype: histories (relative)
and loadings (absolute and relative to the largest loading).  Sizes the
tolerances of the GPU parity suites."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]

import paper_1312_6182_b200 as gps  # noqa: E402
from golden_cases import case_matrix, dense_z, load_solves  # noqa: E402


def main():
    worst = {}
    for case in load_solves():
        if "rank_error" in case:
            continue
        A = case_matrix(case)
        for dt in (np.float64, np.float32):
            D = gps.DataMatrix(A.astype(dt), dtype=dt)
            kw = dict(case["config"])
            if case["solver"] == "single_unit":
                z, r = gps.solve_single_unit(D, gps.SolverConfig(penalty=case["penalty"], gamma=case["gamma"], **kw))
                hist, hist_ref = [r.objective_history], [case["history"]]
            elif case["solver"] == "multi_sequential":
                z, r = gps.solve_multi_sequential(D, gps.SolverConfig(penalty=case["penalty"], gamma=case["gamma"],
                                                                      m=case["m"], **kw))
                hist, hist_ref = r.component_histories, case["histories"]
            else:
                z, r = gps.solve_block(D, gps.SolverConfig(penalty=case["penalty"], mode="block", m=case["m"],
                                                           gamma=case["gamma"], mu=case["mu"], **kw))
                hist, hist_ref = [r.objective_history], [case["history"]]
            Zg = dense_z(case, A.shape[1])
            its = r.iterations == case["iterations"]
            hrel = max((np.max(np.abs(np.array(h) - np.array(g)) / np.maximum(np.abs(g), 1e-300))
                        if len(h) == len(g) else np.inf) for h, g in zip(hist, hist_ref))
            zabs = float(np.max(np.abs(z.values - Zg)))
            sup = bool(np.array_equal(z.values != 0, Zg != 0))
            key = f"{case['name']}[{np.dtype(dt).name}]"
            print(f"{key:40s} iters_equal={its} support_equal={sup} hist_rel={hrel:.2e} z_abs={zabs:.2e}", flush=True)
            worst[np.dtype(dt).name] = max(worst.get(np.dtype(dt).name, 0.0), hrel, zabs)
    print("worst:", worst)


if __name__ == "__main__":
    main()

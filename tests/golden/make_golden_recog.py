"""Golden fixtures for the recognition path, produced by running the
REFERENCE (`gpspca.pca`, `gpspca.datasets`) in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_recog.py

Inputs are recipes (PCG64 seeds); outputs go to tests/golden/recog.json.
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import gpspca  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from recipes import knn_case, recog_samples as samples, sparse_loadings  # noqa: E402


def main():
    out = {"projection": [], "knn": []}
    for seed, (n, f, m) in enumerate([(60, 40, 4), (200, 33, 6), (17, 90, 3)]):
        S = samples(100 + seed, n, f)
        model = gpspca.pca_fit(S, m)
        L = sparse_loadings(200 + seed, f, m + 1, max(2, f // 5))
        mean_given = S[: n // 2].mean(axis=0)
        out["projection"].append({
            "seed": 100 + seed, "loading_seed": 200 + seed, "n": n, "f": f, "m": m,
            "pca_components": model.components.tolist(),
            "pca_singular_values": model.singular_values.tolist(),
            "pca_mean": model.mean.tolist(),
            "project_pca": gpspca.project(S, model.components).tolist(),
            "project_sparse": gpspca.project(S, L).tolist(),
            "project_sparse_given_mean": gpspca.project(S, L, mean=mean_given).tolist(),
            "ev_pca": gpspca.explained_variance(S, model.components).tolist(),
            "ev_sparse": gpspca.explained_variance(S, L).tolist(),
        })
    for seed, (r, t, dim, nl, dup) in enumerate([(40, 25, 5, 4, True), (300, 120, 12, 7, False), (8, 6, 2, 3, True)]):
        train, labels, test = knn_case(300 + seed, r, t, dim, nl, dup)
        case = {"seed": 300 + seed, "r": r, "t": t, "dim": dim, "n_labels": nl, "dup": dup, "pred": {}}
        for k in (1, 2, 3, 5):
            if k <= r:
                pred, _ = gpspca.knn_classify(train, labels, test, k=k)
                case["pred"][str(k)] = pred.tolist()
        out["knn"].append(case)
    with open(os.path.join(HERE, "recog.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote recog.json")


if __name__ == "__main__":
    main()

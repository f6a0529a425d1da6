"""Loader helpers for tests/golden/*.json (reference outputs)."""

import json
import os

import numpy as np

from recipes import digest, make_matrix

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_solves():
    with open(os.path.join(HERE, "solves.json")) as fh:
        return json.load(fh)["cases"]


def load_kernels():
    with open(os.path.join(HERE, "kernels.json")) as fh:
        return json.load(fh)


def case_matrix(case):
    A = make_matrix(case["recipe"])
    assert digest(A) == case["sha"], "input generator drifted from the golden fixture"
    return A


def dense_z(case, n):
    cols = case["z"]
    Z = np.zeros((n, len(cols)))
    for j, col in enumerate(cols):
        Z[col["idx"], j] = col["val"]
    return Z

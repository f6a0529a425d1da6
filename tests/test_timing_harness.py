"""Timing harness: CSV schema on CPU, device run on GPU
checked row by row against the oracle's iteration counts."""

import numpy as np
import pytest

import oracle
from paper_1312_6182_b200.timing import TimingConfig, emit_report, fit_projection, run_timing_experiment


def test_emit_report_schema(tmp_path):
    rows = [{"variant": "sl1", "N": 500, "P": 50, "gamma": 0.01, "workers": 1, "instance": 0,
             "seconds": 0.1, "iterations": 7},
            {"variant": "sl1", "N": 500, "P": 50, "gamma": 0.01, "workers": 1, "instance": "median",
             "seconds": 1 / 3, "iterations": 7.0}]
    path = tmp_path / "t.csv"
    emit_report(rows, str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == "variant,N,P,gamma,workers,instance,seconds,iterations"
    assert lines[2].split(",")[6] == f"{1 / 3:.17g}"
    with pytest.raises(ValueError):
        emit_report([], str(path))
    with pytest.raises(ValueError):
        emit_report([rows[0], {"x": 1}], str(path))


def test_config_validation():
    with pytest.raises(ValueError):
        TimingConfig(m=0)
    with pytest.raises(ValueError):
        TimingConfig(timing_variants=("pca",))
    assert TimingConfig(m=5).m == (5,)
    with pytest.raises(ValueError):
        fit_projection(np.zeros((3, 3)), "pca", 1, 0.1)


@pytest.mark.gpu
def test_device_timing_sweep_matches_oracle(tmp_path):
    cfg = TimingConfig(m=(5,), seed=9, out=str(tmp_path / "timing.csv"), timing_sizes=(500, 1000),
                       timing_gammas=(0.01, 0.05), timing_instances=2, max_iter=200)
    rows = run_timing_experiment(cfg)
    text = (tmp_path / "timing.csv").read_text().splitlines()
    assert text[0] == "variant,N,P,gamma,workers,instance,seconds,iterations"
    assert len(text) == 1 + len(rows) == 1 + 2 * 4 * 2 * 3
    for r in rows:
        if r["instance"] == "median":
            continue
        A = np.random.default_rng([9, r["N"], r["instance"]]).standard_normal((r["P"], r["N"]))
        pen = "l1" if r["variant"].endswith("1") else "l0"
        if r["variant"].startswith("s"):
            _, hists, _ = oracle.multi_sequential(A, [r["gamma"]] * 5, pen, max_iter=200)
            iters = sum(len(h) - 1 for h in hists)
        else:
            _, hist, _, _ = oracle.block_solve(A, 5, r["gamma"], 1.0, pen, max_iter=200,
                                               init="random_orthonormal", seed=[9, r["N"], r["instance"]])
            iters = len(hist) - 1
        assert r["iterations"] == iters, r

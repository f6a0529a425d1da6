"""Timing harness on the device (reference bench.py:219-298).

`run_timing_experiment` sweeps the paper's size grid (P = N/10)
over the four GP-SPCA variants exactly as the reference's timing sweep does
-- same instance seeds (default_rng([seed, N, instance]), bench.py:245-246),
same solvers (solve_multi_sequential for sl*, solve_block with
random_orthonormal init for bl*, bench.py:102-113), same CSV schema
`variant,N,P,gamma,workers,instance,seconds,iterations` with per-cell median
rows -- but every solve runs on the B200 engine.  `device_columns=True`
appends `device,n_gpus` for side-by-side CPU/GPU tables.  The recognition
experiment (PCA baseline, datasets, k-NN) is outside this path's scope.
"""

import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .block import solve_block
from .core import DataMatrix, SolverConfig, center_columns_with_means
from .single_unit import solve_multi_sequential

SPCA_VARIANTS = ("sl1", "sl0", "bl1", "bl0")


@dataclass
class TimingConfig:
    """The reference ExperimentConfig (bench.py:34-75) as far as the timing
    sweep reads it.  The recognition-experiment fields (dataset, split,
    knn_k, ...) and the CPU-plan fields (workers, chunk, timing_workers) are
    accepted so reference call sites construct it unchanged; the device
    ignores the plan (one GPU, fixed grid) and reports workers = 1."""

    dataset: str = None
    format: str = "csv_labeled"
    variant: str = "sl1"
    m: tuple = (5,)
    gamma: float = 0.1
    repetitions: int = 1
    workers: int = 1
    chunk: int = 256
    knn_k: int = 1
    split: object = None
    report_timing: bool = True
    timing_workers: tuple = None
    mu: float = 1.0
    seed: int = 0
    out: str = None
    tol: float = 1e-6
    max_iter: int = 1000
    timing_sizes: tuple = (500, 1000, 2000)
    timing_gammas: tuple = (0.01, 0.05)
    timing_variants: tuple = SPCA_VARIANTS
    timing_instances: int = 20
    device_columns: bool = False
    warmup: bool = True  # untimed solve per variant first (device start-up is not per-solve cost)

    def __post_init__(self):
        if isinstance(self.m, int):
            self.m = (self.m,)
        self.m = tuple(int(v) for v in self.m)
        if any(v < 1 for v in self.m):
            raise ValueError("m values must be >= 1")
        if self.timing_instances < 1:
            raise ValueError("timing_instances must be >= 1")
        bad = [v for v in self.timing_variants if v not in SPCA_VARIANTS]
        if bad:
            raise ValueError(f"unknown variants {bad}; expected a subset of {SPCA_VARIANTS}")


def fit_projection(train_samples, variant, m, gamma, mu=1.0, tol=1e-6, max_iter=1000, seed=0, center=True):
    """SPCA variants of reference bench.py:78-114 on the device; returns
    (loadings n x m, feature means, RunReport)."""
    if variant not in SPCA_VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    A = DataMatrix(np.asarray(train_samples, dtype=np.float64))
    if center:  # on the device: column means and the centred copy (core.py:234-240)
        A, mean = center_columns_with_means(A)
    else:
        mean = np.zeros(A.n)
    penalty = "l1" if variant.endswith("1") else "l0"
    if variant.startswith("s"):
        cfg = SolverConfig(penalty=penalty, mode="single_unit", m=m, gamma=gamma, mu=mu, tol=tol,
                           max_iter=max_iter, seed=seed)
        loadings, report = solve_multi_sequential(A, cfg)
    else:
        cfg = SolverConfig(penalty=penalty, mode="block", m=m, gamma=gamma, mu=mu, tol=tol, max_iter=max_iter,
                           init="random_orthonormal", seed=seed)
        loadings, report = solve_block(A, cfg)
    return loadings.values, mean, report


def run_timing_experiment(config):
    """Wall-time sweep over random dense instances on the (N, P = N/10) grid
    (reference bench.py:219-269); returns the rows (and writes config.out)."""
    m = config.m[0]
    rows = []
    dev = _native.default_device()
    if config.warmup:  # one untimed solve per variant: CUDA context, graphs, first launches
        N0 = min(config.timing_sizes)
        A0 = np.random.default_rng([config.seed, N0, 0]).standard_normal((N0 // 10, N0))
        for variant in config.timing_variants:
            fit_projection(A0, variant, m, config.timing_gammas[0], config.mu, config.tol, config.max_iter,
                           seed=[config.seed, N0, 0], center=False)
    for N in sorted(config.timing_sizes):
        if N % 10:
            raise ValueError(f"size {N} violates the P = N/10 grid")
        P = N // 10
        for variant in config.timing_variants:
            for gamma in config.timing_gammas:
                seconds, iterations = [], []
                for instance in range(config.timing_instances):
                    rng = np.random.default_rng([config.seed, N, instance])
                    A = rng.standard_normal((P, N))
                    start = time.perf_counter()
                    _, _, report = fit_projection(A, variant, m, gamma, config.mu, config.tol, config.max_iter,
                                                  seed=[config.seed, N, instance], center=False)
                    elapsed = time.perf_counter() - start
                    seconds.append(elapsed)
                    iterations.append(report.iterations)
                    row = {"variant": variant, "N": N, "P": P, "gamma": gamma, "workers": 1,
                           "instance": instance, "seconds": elapsed, "iterations": report.iterations}
                    if config.device_columns:
                        row.update(device=f"cuda:{dev}", n_gpus=1)
                    rows.append(row)
                med = {"variant": variant, "N": N, "P": P, "gamma": gamma, "workers": 1, "instance": "median",
                       "seconds": float(np.median(seconds)), "iterations": float(np.median(iterations))}
                if config.device_columns:
                    med.update(device=f"cuda:{dev}", n_gpus=1)
                rows.append(med)
    if config.out:
        emit_report(rows, config.out)
    return rows


def emit_report(rows, path):
    """UTF-8 CSV, LF endings, 17-significant-digit floats (bench.py:272-298)."""
    if not rows:
        raise ValueError("nothing to report")
    fields = list(rows[0].keys())
    for i, row in enumerate(rows):
        if list(row.keys()) != fields:
            raise ValueError(f"row {i} does not match the header {fields}")
    with open(path, "w", encoding="utf-8", newline="") as fh:
        fh.write(",".join(fields) + "\n")
        for row in rows:
            fh.write(",".join(_field(row[k]) for k in fields) + "\n")


def _field(value):
    if value is None:
        return ""
    if isinstance(value, (float, np.floating)):
        return f"{float(value):.17g}"
    if isinstance(value, (int, np.integer)):
        return str(int(value))
    text = str(value)
    if "," in text or '"' in text or "\n" in text:
        text = '"' + text.replace('"', '""') + '"'
    return text

"""Support refinement for single-unit solves (reference single_unit.py:213-264).

Off by default (core.py:178-179).  When enabled, the converged support is
perturbed by relaxing / tightening gamma, the leading direction of each
perturbed support is found by power iteration on the GATHERED columns
(a small device matrix: `gps_matrix_gather`), and the full device power
loop is re-run from it; any strict improvement is kept.
"""

import numpy as np

from . import _native
from .core import DataMatrix
from .parallel import par_gram_apply, par_matvec_t


def _active(c, gamma, penalty):
    return np.abs(c) > gamma if penalty == "l1" else c * c > gamma


def _identity(v):
    return v


def restricted_leading_direction(A, support, x, iters=50, project=None):
    """Leading left singular direction of A[:, support] by power iteration
    seeded at x (single_unit.py:219-230); None when it collapses to 0.

    With `project` (the implicit-deflation projector P = I - XX' of
    solve_multi_sequential) the restricted matrix is the deflated one,
    (PA)[:, S] = P A_S, so each step is v <- P A_S A_S' P v: the reference
    gathers the columns of the explicitly deflated matrix
    (single_unit.py:222, :287-296, :320-330)."""
    project = project or _identity
    idx = np.ascontiguousarray(np.flatnonzero(support), dtype=np.int64)
    h = _native.C.c_void_p()
    _native.check(_native.lib().gps_matrix_gather(
        A.handle, idx.ctypes.data_as(_native._i64p), idx.size, _native.C.byref(h)))
    sub = DataMatrix._wrap(A.context, h)
    v = np.array(x, dtype=np.float64)
    for _ in range(iters):
        v = project(par_gram_apply(sub, par_matvec_t(sub, project(v))))
        nrm = np.linalg.norm(v)
        if nrm == 0.0:
            return None
        v = v / nrm
    return v


def refine_support(A, best, gamma, config, loop, project=None):
    """single_unit.py:233-264 on the device; best = (x, history, converged, w).

    `project` is the deflation projector of a later solve_multi_sequential
    component: the correlations are those of the deflated matrix,
    (PA)'x = A'(Px), and every restart direction lies in range(P), which
    the loop's deflated sweeps keep it in."""
    if gamma <= 0:
        return best
    project = project or _identity
    x, history, converged, w = best
    for _ in range(4):
        c = par_matvec_t(A, project(x))
        current = _active(c, gamma, config.penalty)
        improved = False
        for delta in (0.02, 0.05, 0.1, 0.2, 0.4):
            for g2 in (gamma * (1.0 - delta), gamma * (1.0 + delta)):
                support = _active(c, g2, config.penalty)
                if not support.any() or np.array_equal(support, current):
                    continue
                x0 = restricted_leading_direction(A, support, x, project=project)
                if x0 is None:
                    continue
                trial = loop.run(x0)
                if trial[1][-1] > history[-1] * (1.0 + 1e-12):
                    best = trial  # keeps the trial's near-threshold list (.band)
                    x, history, converged, w = trial
                    improved = True
        if not improved:
            break
    return best

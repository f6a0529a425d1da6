"""CPU oracle for the GP-SPCA hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain NumPy fp64, the algorithm of the reference
package `gpspca` 0.1.0 (`/root/reference/pkg/src/gpspca`) for the power
iteration path only.  It exists to check the CUDA engine, never to be it:
only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg
(and `bench.py --impl reference`) may import it.  The product package
`paper_1312_6182_b200` never imports anything from here and fails loudly if
its CUDA library is missing.

Parity status: PINNED.  `tests/golden/*.json` were produced by running the
reference itself in the build container (`tests/golden/make_golden.py`,
`tests/golden/make_golden_recog.py`); `tests/test_oracle_golden.py` and
`tests/test_recognition.py` check these restatements against them.

`oracle.recognition` restates the recognition path around the solver
(projection, explained variance, k-NN, dense PCA).
"""

from .gpower import *  # noqa: F401,F403
from .gpower import __all__  # noqa: F401

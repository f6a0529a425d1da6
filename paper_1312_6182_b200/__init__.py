"""B200-native GP-SPCA engine: a drop-in for the power-iteration path of the
reference `gpspca` package (sparse PCA by the generalized power method,
arXiv:1312.6182).

Same public names, signatures and exceptions as the reference API
(`/root/reference/pkg/src/gpspca/__init__.py:8-69`) for the hot path:
single-unit l1/l0 and block l1/l0 solvers, their one-shot objectives /
ascent directions / recovery, the column kernel seam, and the recognition
path around them (project, explained_variance, knn_classify, pca_fit).  Arithmetic runs in
hand-written sm_100a CUDA (libgpspca_b200.so, include/gpspca_b200.h); there is
no CPU fallback.
"""

from .core import (
    DataMatrix,
    RunReport,
    SolverConfig,
    SparseLoadings,
    StiefelPoint,
    as_data_matrix,
    center_columns,
    column_norms,
    gram_quadratic,
    positive_part,
)
from .parallel import (
    DEFAULT_PLAN,
    KernelPlan,
    fused_sweep,
    par_gram_apply,
    par_matvec_t,
    par_threshold_accumulate,
    threshold_weights,
)
from .single_unit import (
    SingleUnitState,
    ascent_direction_sl0,
    ascent_direction_sl1,
    deflate,
    objective_sl0,
    objective_sl1,
    power_step,
    recover_pattern_sl0,
    recover_pattern_sl1,
    solve_multi_sequential,
    solve_single_unit,
)
from .timing import TimingConfig, emit_report, fit_projection, run_timing_experiment
from .timing import TimingConfig as ExperimentConfig
from .recognition import PcaModel, deterministic_signs, explained_variance, knn_classify, pca_fit, project
from .block import (
    BlockState,
    RankDeficiencyError,
    ascent_direction_block,
    objective_bl0,
    objective_bl1,
    polar_projection,
    solve_block,
)

__version__ = "0.1.0+b200"

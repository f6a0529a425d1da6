"""Block sparse PCA (l1 / l0) on the Stiefel manifold (reference block.py).
Device implementation lands with the block sweep kernels."""

from dataclasses import dataclass

from .core import StiefelPoint


@dataclass(frozen=True)
class BlockState:
    """Stiefel iterate, objective, step count (block.py:20-30)."""

    X: StiefelPoint
    objective: float
    iteration: int


class RankDeficiencyError(RuntimeError):
    """Gradient lost full column rank (block.py:33-49)."""

    def __init__(self, rank, required, iteration=None):
        self.rank = rank
        self.required = required
        self.iteration = iteration
        where = "" if iteration is None else f" at iteration {iteration}"
        super().__init__(f"gradient has numerical rank {rank} < {required}{where}; reduce gamma or m")


def _todo(*a, **k):
    raise NotImplementedError("block path not built yet")


objective_bl1 = objective_bl0 = ascent_direction_block = polar_projection = solve_block = _todo

"""Gaussian-RBF grid of the influence functions (drop-in for
specklediff.influence.RbfGrid, reference influence.py:9-37).

The evaluation phi_i(z) = sum_j w_ij exp(-(z - mu_j)^2 / (2 gamma^2)) itself
happens inside the fused stage kernel (csrc/tnrd_stage.cuh).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RbfGrid:
    """count equispaced centres on [-radius, radius]; gamma defaults to the
    centre spacing (influence.py:33-37)."""

    count: int
    radius: float
    bandwidth: float | None = None

    def __post_init__(self):
        if self.count < 2:
            raise ValueError("need at least 2 RBF centers")
        if not self.radius > 0:
            raise ValueError("radius must be positive")
        if self.bandwidth is not None and not self.bandwidth > 0:
            raise ValueError("bandwidth must be positive")

    @property
    def spacing(self) -> float:
        return 2.0 * self.radius / (self.count - 1)

    @property
    def centers(self) -> np.ndarray:
        return np.linspace(-self.radius, self.radius, self.count)

    @property
    def gamma(self) -> float:
        return self.spacing if self.bandwidth is None else float(self.bandwidth)

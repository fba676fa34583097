"""Speckle data term (drop-in for the hot-path parts of specklediff.speckle).

* ``prox_idiv`` -- closed-form I-divergence prox (speckle.py:103-121), GPU.
* ``SpeckleConfig`` / ``speckle_field`` / ``sample_speckle`` -- the
  reference's Philox-keyed L-look amplitude speckle (speckle.py:24-70),
  restated on the host.  It is the INPUT GENERATOR for the synthetic
  benchmark configs (BASELINE.json), not part of the accelerated path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import require_cuda, torch, _stream_handle, _ptr
from .imageops import as_image

GENERATOR_NAME = "philox"
F_FLOOR = 1e-6  # speckle.py:21


@dataclass(frozen=True)
class SpeckleConfig:
    looks: int
    seed: int

    def __post_init__(self):
        if self.looks < 1:
            raise ValueError(f"looks must be >= 1, got {self.looks}")
        if not 0 <= int(self.seed) < 2 ** 64:
            raise ValueError("seed must fit in an unsigned 64-bit integer")


@dataclass(frozen=True)
class NoisyPair:
    clean: np.ndarray
    noisy: np.ndarray
    config: SpeckleConfig

    def __post_init__(self):
        if self.clean.shape != self.noisy.shape:
            raise ValueError("clean and noisy images must share dimensions")


def speckle_field(shape, cfg: SpeckleConfig) -> np.ndarray:
    """Amplitude speckle sqrt(Gamma(L, 1/L)) from a Philox generator keyed
    by the seed (speckle.py:51-61), bit-identical to the reference."""
    gen = np.random.Generator(np.random.Philox(key=int(cfg.seed)))
    return np.sqrt(gen.gamma(shape=float(cfg.looks), scale=1.0 / cfg.looks,
                             size=shape))


def sample_speckle(u, cfg: SpeckleConfig) -> NoisyPair:
    """speckle.py:64-70"""
    u = as_image(u, "clean image")
    if (u < 0).any():
        raise ValueError("clean image must be nonnegative")
    return NoisyPair(clean=u, noisy=u * speckle_field(u.shape, cfg), config=cfg)


def prox_idiv(u_tilde, f, lam: float) -> np.ndarray:
    """argmin_u |u - u~|^2/2 + lam <u^2 - 2 f^2 log u, 1>, pointwise
    (u~ + sqrt(u~^2 + 8 a lam f^2)) / (2a), a = 1 + 2 lam, f >= 1e-6
    (speckle.py:103-121); evaluated on the GPU in fp32."""
    if not lam > 0:
        raise ValueError(f"lambda must be positive, got {lam}")
    u_tilde = as_image(u_tilde, "u_tilde")
    f = as_image(f, "f")
    u_tilde, f = np.broadcast_arrays(u_tilde, f)
    require_cuda()
    t = torch()
    ut = t.from_numpy(np.ascontiguousarray(u_tilde, dtype=np.float32)).cuda()
    ft = t.from_numpy(np.ascontiguousarray(f, dtype=np.float32)).cuda()
    out = t.empty_like(ut)
    _lib.check(_lib.load().tnrd_prox_idiv(_ptr(ut), _ptr(ft), _ptr(out),
                                          ut.numel(), float(lam),
                                          _stream_handle()))
    return out.cpu().numpy().astype(np.float64)

"""Speckle data term (drop-in for the hot-path parts of specklediff.speckle).

* ``prox_idiv`` -- closed-form I-divergence prox (speckle.py:103-121), GPU.
* ``SpeckleConfig`` / ``speckle_field`` / ``sample_speckle`` -- the
  reference's Philox-keyed L-look amplitude speckle (speckle.py:24-70),
  restated on the host, bit-identical to the reference.  It is the INPUT
  GENERATOR for the synthetic benchmark configs (BASELINE.json).
* ``speckle_field_device`` / ``sample_speckle_device`` / ``sample_speckle_gpu``
  -- the same distribution generated on the GPU (tnrd_sample_speckle:
  counter-based Philox4x32-10 + Marsaglia-Tsang).
  Equal to the reference in distribution, not bitwise: numpy's sequential
  rejection stream has no parallel equivalent.
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


def nakagami_mean(looks: int) -> float:
    """E[n] of the unit-power amplitude speckle (speckle.py:73-75):
    Gamma(L + 1/2) / (Gamma(L) sqrt(L))."""
    import math
    return math.gamma(looks + 0.5) / (math.gamma(looks) * math.sqrt(looks))


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


# ------------------------------------------------------------------ GPU

def _seed_u64(cfg: SpeckleConfig) -> int:
    return int(cfg.seed) & 0xFFFFFFFFFFFFFFFF


def sample_speckle_device(clean, cfg: SpeckleConfig, out=None, stream=None,
                          check: bool = True):
    """noisy = clean * n on the GPU for a CUDA fp32 tensor (H, W) or
    (B, H, W) (tnrd_sample_speckle).  Pixel (b, y, x) draws from counter
    index b*H*W + y*W + x, so a batch equals its images generated with the
    matching index offsets, for any launch geometry.  ``clean=None`` is not
    accepted here; see speckle_field_device."""
    from .engine import stream_ctx
    with stream_ctx(stream):
        return _sample_speckle_device(clean, cfg, out, check)


def _sample_speckle_device(clean, cfg, out, check):
    from .engine import Status
    t = torch()
    require_cuda()
    if clean.dtype != t.float32 or not clean.is_cuda:
        raise ValueError("clean must be a CUDA float32 tensor")
    if clean.dim() not in (2, 3):
        raise ValueError(f"expected (H, W) or (B, H, W), got {tuple(clean.shape)}")
    clean = clean if clean.stride(-1) == 1 else clean.contiguous()
    B, H, W = (1, *clean.shape) if clean.dim() == 2 else tuple(clean.shape)
    if out is None:
        out = t.empty_strided(clean.shape, clean.stride(), dtype=t.float32, device=clean.device)
    if out.shape != clean.shape or out.stride() != clean.stride():
        raise ValueError("out must match clean's shape and strides")
    ld = clean.stride(-2)
    img_stride = clean.stride(0) if clean.dim() == 3 else ld * H
    st = Status(clean.device) if check else None
    if st is not None:
        st.reset()
    _lib.check(_lib.load().tnrd_sample_speckle(
        _ptr(clean), _ptr(out), B, H, W, ld, img_stride, int(cfg.looks),
        _seed_u64(cfg), _ptr(st.buf) if st is not None else None,
        _stream_handle()))
    if st is not None:
        host = st.buf.cpu().numpy().view(np.uint32)
        if host[1] != 0xFFFFFFFF:
            raise ValueError("clean image must be nonnegative and finite")
    return out


def speckle_field_device(shape, cfg: SpeckleConfig, device=None, stream=None):
    """The amplitude speckle field n (fp32, shape (H, W) or (B, H, W)) on
    the GPU: sqrt(Gamma(L, 1/L)) per pixel."""
    from .engine import stream_ctx
    with stream_ctx(stream):
        return _speckle_field_device(shape, cfg, device)


def _speckle_field_device(shape, cfg, device):
    t = torch()
    require_cuda()
    shape = tuple(int(v) for v in shape)
    if len(shape) not in (2, 3) or min(shape) < 1:
        raise ValueError(f"bad field shape {shape}")
    out = t.empty(shape, dtype=t.float32, device=device or "cuda")
    B, H, W = (1, *shape) if len(shape) == 2 else shape
    _lib.check(_lib.load().tnrd_sample_speckle(
        None, _ptr(out), B, H, W, W, H * W, int(cfg.looks), _seed_u64(cfg),
        None, _stream_handle()))
    return out


def sample_speckle_gpu(u, cfg: SpeckleConfig) -> NoisyPair:
    """sample_speckle (speckle.py:64-70) with the field drawn on the GPU;
    same validation and NoisyPair (float64 arrays) as the reference."""
    u = as_image(u, "clean image")
    if (u < 0).any():
        raise ValueError("clean image must be nonnegative")
    t = torch()
    require_cuda()
    dev = t.from_numpy(np.ascontiguousarray(u, dtype=np.float32)).cuda()
    noisy = sample_speckle_device(dev, cfg, check=False)
    return NoisyPair(clean=u, noisy=noisy.cpu().numpy().astype(np.float64), config=cfg)

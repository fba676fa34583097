"""Seeded synthetic workloads of BASELINE.json (configs C1..C5).

The reference ships no image generator or dataset for its benchmark; these
stand-ins follow BASELINE.json's description:
  * clean images: piecewise-smooth fields of random rectangles/ellipses,
    each a base level plus a linear ramp, clipped to [1, 255];
  * observation f = clean x amplitude speckle sqrt(Gamma(L, 1/L)) from the
    reference's own Philox-keyed sampler (speckle.sample_speckle);
  * model: per stage coeffs ~ N(0,1) row-normalised (zero-mean, unit-L2
    kernels since the basis is orthonormal), RBF weights ~ N(0, 0.1^2) on
    RbfGrid(63, 310) (gamma = 10), beta = 0 (lambda = 1) -- the convention of
    the reference's tests/test_diffusion.py:12-22.
Seeds: model = config index; clean image = 1000*cfg + image index; speckle =
10**6 + 1000*cfg + image index; C4 scene tiles use (cfg, tile_row, tile_col).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .diffusion import DiffusionModel, StageParams
from .influence import RbfGrid
from .speckle import SpeckleConfig, sample_speckle


@dataclass(frozen=True)
class Config:
    name: str
    index: int
    H: int
    W: int
    batch: int
    m: int
    nk: int
    T: int
    looks: tuple
    M: int = 63
    tiled: bool = False
    note: str = ""

    def looks_for(self, i: int) -> int:
        return self.looks[i % len(self.looks)]

    @property
    def pixels(self) -> int:
        return self.batch * self.H * self.W


CONFIGS = {
    "c1": Config("c1", 1, 256, 256, 1, 5, 24, 5, (1,),
                 note="TNRD 5x5, Nk=24, 5 stages, one 256x256 image, L=1"),
    "c2": Config("c2", 2, 512, 512, 1, 7, 48, 5, (4,),
                 note="TNRD 7x7, Nk=48, 5 stages, one 512x512 image, L=4 "
                      "(single-image latency case)"),
    "c3": Config("c3", 3, 512, 512, 256, 7, 48, 5, (1, 2, 4, 8),
                 note="TNRD 7x7, Nk=48, 5 stages, 256 x 512x512, L cycles "
                      "1,2,4,8"),
    "c4": Config("c4", 4, 16384, 16384, 1, 7, 48, 5, (1,), tiled=True,
                 note="TNRD 7x7, Nk=48, 5 stages, one 16384x16384 tiled "
                      "scene, L=1"),
    "c5": Config("c5", 5, 1024, 1024, 32, 9, 80, 8, (2,),
                 note="TNRD 9x9, Nk=80, 8 stages, 32 x 1024x1024, L=2"),
}


def make_model(m: int, nk: int, T: int, M: int = 63, seed: int = 0,
               weight_scale: float = 0.1, beta: float = 0.0,
               radius: float = 310.0, looks: int = 1) -> DiffusionModel:
    rng = np.random.default_rng(seed)
    stages = []
    for _ in range(T):
        c = rng.standard_normal((nk, m * m - 1))
        c /= np.linalg.norm(c, axis=1, keepdims=True)
        w = weight_scale * rng.standard_normal((nk, M))
        stages.append(StageParams(beta=beta, coeffs=c, weights=w))
    return DiffusionModel(stages=stages, filter_size=m, looks=looks,
                          value_range=255.0, rbf=RbfGrid(M, radius),
                          variant="prox", seed=seed)


def config_model(cfg: Config) -> DiffusionModel:
    return make_model(cfg.m, cfg.nk, cfg.T, cfg.M, seed=cfg.index,
                      looks=cfg.looks[0])


def clean_image(H: int, W: int, seed, n_shapes: int | None = None) -> np.ndarray:
    """Piecewise-smooth [1, 255] float64 field."""
    rng = np.random.default_rng(seed)
    ys = (np.arange(H) + 0.5) / H
    xs = (np.arange(W) + 0.5) / W
    Y, X = np.meshgrid(ys, xs, indexing="ij")
    g = rng.uniform(-60.0, 60.0, 2)
    img = rng.uniform(60.0, 200.0) + g[0] * (Y - 0.5) + g[1] * (X - 0.5)
    if n_shapes is None:
        n_shapes = int(rng.integers(10, 22))
    for _ in range(n_shapes):
        cy, cx = rng.uniform(0.0, 1.0, 2)
        hy, hx = rng.uniform(0.04, 0.3, 2)
        level = rng.uniform(1.0, 255.0)
        gy, gx = rng.uniform(-120.0, 120.0, 2)
        if rng.integers(2) == 0:
            mask = (np.abs(Y - cy) < hy) & (np.abs(X - cx) < hx)
        else:
            mask = ((Y - cy) / hy) ** 2 + ((X - cx) / hx) ** 2 < 1.0
        img = np.where(mask, level + gy * (Y - cy) + gx * (X - cx), img)
    return np.clip(img, 1.0, 255.0)


def noisy_image(cfg: Config, index: int, H: int | None = None,
                W: int | None = None):
    """(clean, f) for image ``index`` of a batch config, f rounded to fp32
    (the handoff both the GPU path and the oracle see)."""
    H = cfg.H if H is None else H
    W = cfg.W if W is None else W
    clean = clean_image(H, W, 1000 * cfg.index + index)
    pair = sample_speckle(clean, SpeckleConfig(
        looks=cfg.looks_for(index), seed=10 ** 6 + 1000 * cfg.index + index))
    return clean, pair.noisy.astype(np.float32)


SCENE_TILE = 1024


def scene_tile(cfg: Config, tr: int, tc: int):
    """Tile (tr, tc) of the tiled scene (C4): independent seeds so any crop
    can be regenerated without the whole scene."""
    seed = np.random.SeedSequence([cfg.index, tr, tc]).generate_state(2)
    clean = clean_image(SCENE_TILE, SCENE_TILE, seed)
    s = int(np.random.SeedSequence([10 ** 6, cfg.index, tr, tc])
            .generate_state(1, dtype=np.uint64)[0])
    pair = sample_speckle(clean, SpeckleConfig(looks=cfg.looks[0], seed=s))
    return clean, pair.noisy.astype(np.float32)


def scene_rows(cfg: Config, row0: int, row1: int, with_clean: bool = False):
    """Rows [row0, row1) of the tiled scene (fp32 noisy, optionally clean)."""
    T = SCENE_TILE
    nt = cfg.W // T
    f = np.empty((row1 - row0, cfg.W), dtype=np.float32)
    c = np.empty((row1 - row0, cfg.W), dtype=np.float64) if with_clean else None
    for tr in range(row0 // T, (row1 - 1) // T + 1):
        a, b = max(row0, tr * T), min(row1, (tr + 1) * T)
        for tc in range(nt):
            cl, fn = scene_tile(cfg, tr, tc)
            f[a - row0:b - row0, tc * T:(tc + 1) * T] = fn[a - tr * T:b - tr * T]
            if with_clean:
                c[a - row0:b - row0, tc * T:(tc + 1) * T] = cl[a - tr * T:b - tr * T]
    return (f, c) if with_clean else f


def scene_crop(cfg: Config, y0: int, y1: int, x0: int, x1: int) -> np.ndarray:
    """Noisy fp32 crop [y0:y1, x0:x1] of the tiled scene."""
    T = SCENE_TILE
    out = np.empty((y1 - y0, x1 - x0), dtype=np.float32)
    for tr in range(y0 // T, (y1 - 1) // T + 1):
        for tc in range(x0 // T, (x1 - 1) // T + 1):
            _, fn = scene_tile(cfg, tr, tc)
            a, b = max(y0, tr * T), min(y1, (tr + 1) * T)
            c, d = max(x0, tc * T), min(x1, (tc + 1) * T)
            out[a - y0:b - y0, c - x0:d - x0] = fn[a - tr * T:b - tr * T,
                                                   c - tc * T:d - tc * T]
    return out


# ---- parallel generation (host cores; numpy work per image / scene tile) ----

def _pool(workers):
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    import os
    n = workers or min(32, os.cpu_count() or 1)
    # fork: children only run numpy (call before any CUDA work in the parent
    # where possible; they never touch the device)
    return ProcessPoolExecutor(max_workers=n, mp_context=mp.get_context("fork")), n


def _noisy_f(args):
    cfg, i = args
    return noisy_image(cfg, i)[1]


def noisy_batch(cfg: Config, indices, workers: int | None = None) -> np.ndarray:
    """fp32 observations of images ``indices`` of a batch config, stacked
    (B, H, W); generated on all host cores (bit-identical to noisy_image)."""
    indices = list(indices)
    if len(indices) <= 2:
        return np.stack([noisy_image(cfg, i)[1] for i in indices])
    ex, _ = _pool(workers)
    with ex:
        return np.stack(list(ex.map(_noisy_f, [(cfg, i) for i in indices])))


def _tile_f(args):
    cfg, tr, tc = args
    return tr, tc, scene_tile(cfg, tr, tc)[1]


def scene_rows_parallel(cfg: Config, row0: int, row1: int, workers: int | None = None) -> np.ndarray:
    """scene_rows(cfg, row0, row1) with the scene tiles generated on all
    host cores (same values)."""
    T = SCENE_TILE
    nt = cfg.W // T
    f = np.empty((row1 - row0, cfg.W), dtype=np.float32)
    jobs = [(cfg, tr, tc) for tr in range(row0 // T, (row1 - 1) // T + 1) for tc in range(nt)]
    ex, _ = _pool(workers)
    with ex:
        for tr, tc, fn in ex.map(_tile_f, jobs):
            a, b = max(row0, tr * T), min(row1, (tr + 1) * T)
            f[a - row0:b - row0, tc * T:(tc + 1) * T] = fn[a - tr * T:b - tr * T]
    return f

"""Parity of the exact paths bench.py times, at the BASELINE sizes.

bench.py runs C3 and C5 as one tnrd_despeckle call over the whole batch in
auto mode (the large-tile fused kernel, batch fork onto two streams) and C4
as the whole 16384^2 scene through tnrd_plan_despeckle_host (row bands on
their own streams, halo rows read in place).  The smaller parity cases in
test_gpu_parity.py reach other kernels (small grids go to the cluster
kernel), so these tests drive the benched launches themselves and compare
with the float64 oracle (SURVEY 8(d) coverage table):

  * C3: all 256 images in one call; images {0..5, 254, 255} (two per looks
    value, first and last index) against the oracle on the full image;
  * C4: tiles of 96^2 at all 4 corners, all 4 edge midpoints, the interior
    and straddling every strip boundary 2048 k (k = 1..7: the G = 2, 4, 8
    boundaries), oracle on tile + T (m - 1) = 30 px margin (the dependency
    radius after T stages: the interior of the margin is exact);
  * C5: all 32 images in one call; image 0 in full against the oracle, plus
    two 192^2 tiles of image 31 (margin T (m - 1) = 64 px).

Bar (north_star): max relative error <= 1e-4, |dPSNR| <= 0.01 dB.
"""
import numpy as np
import pytest

from conftest import parity_stats

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4
PSNR_TOL = 0.01


def _launches_per_stage(fn, T):
    import torch
    torch.cuda.synchronize()
    _lib.launch_count_reset()
    r = fn()
    torch.cuda.synchronize()
    return r, _lib.launch_count() / T


def test_c3_full_batch_benched_path(cuda, oracle):
    torch = cuda
    cfg = synth.CONFIGS["c3"]
    model = synth.config_model(cfg)
    f = torch.from_numpy(synth.noisy_batch(cfg, range(cfg.batch))).cuda()
    dm = tn.device_model_for(model)
    u, per_stage = _launches_per_stage(lambda: dm.despeckle(f), cfg.T)
    # the benched launch: two tile-kernel launches per stage (batch fork)
    assert per_stage == 2, per_stage
    u = u.cpu().numpy()
    for i in (0, 1, 2, 3, 4, 5, 254, 255):
        clean, fi = synth.noisy_image(cfg, i)
        ref = oracle.run_diffusion(fi.astype(np.float64), model)
        st = parity_stats(u[i], ref, clean)
        assert st["rel"] <= REL_TOL and st["dpsnr"] <= PSNR_TOL, (i, st)


C4_TILE = 96


def _c4_positions(N):
    t = C4_TILE
    mid = N // 2 - t // 2
    pos = {"corner_tl": (0, 0), "corner_tr": (0, N - t), "corner_bl": (N - t, 0),
           "corner_br": (N - t, N - t), "edge_top": (0, mid), "edge_bottom": (N - t, mid),
           "edge_left": (mid, 0), "edge_right": (mid, N - t), "interior": (5000, 9000)}
    for k in range(1, 8):   # strip boundaries of G = 8 (k odd), 4 (k = 2, 6), 2 (k = 4)
        pos[f"strip_{2048 * k}"] = (2048 * k - t // 2, (1237 * k) % (N - t))
    return pos


@pytest.fixture(scope="module")
def c4_scene(cuda):
    cfg = synth.CONFIGS["c4"]
    model = synth.config_model(cfg)
    f = synth.scene_rows_parallel(cfg, 0, cfg.H)
    dm = tn.device_model_for(model)
    u = dm.despeckle_host(f)           # tnrd_plan_despeckle_host: banded
    return cfg, model, u


def test_c4_scene_is_banded_and_finite(c4_scene):
    cfg, model, u = c4_scene
    assert u.shape == (cfg.H, cfg.W) and np.all(np.isfinite(u)) and u.min() > 0


@pytest.mark.parametrize("where", list(_c4_positions(16384)))
def test_c4_scene_tiles(c4_scene, oracle, where):
    cfg, model, u = c4_scene
    N, t = cfg.H, C4_TILE
    y, x = _c4_positions(N)[where]
    marg = cfg.T * (cfg.m - 1)
    oy0, oy1 = max(0, y - marg), min(N, y + t + marg)
    ox0, ox1 = max(0, x - marg), min(N, x + t + marg)
    fo = synth.scene_crop(cfg, oy0, oy1, ox0, ox1).astype(np.float64)
    ref = oracle.run_diffusion(fo, model)[y - oy0:y - oy0 + t, x - ox0:x - ox0 + t]
    st = parity_stats(u[y:y + t, x:x + t], ref)
    assert st["rel"] <= REL_TOL, (where, st)


@pytest.fixture(scope="module")
def c5_batch(cuda):
    torch = cuda
    cfg = synth.CONFIGS["c5"]
    model = synth.config_model(cfg)
    f = torch.from_numpy(synth.noisy_batch(cfg, range(cfg.batch))).cuda()
    dm = tn.device_model_for(model)
    u, per_stage = _launches_per_stage(lambda: dm.despeckle(f), cfg.T)
    return cfg, model, u.cpu().numpy(), per_stage


def test_c5_full_image0_benched_path(c5_batch, oracle):
    cfg, model, u, per_stage = c5_batch
    assert per_stage == 2, per_stage      # tile kernel, batch fork
    clean, f0 = synth.noisy_image(cfg, 0)
    ref = oracle.run_diffusion(f0.astype(np.float64), model)
    st = parity_stats(u[0], ref, clean)
    assert st["rel"] <= REL_TOL and st["dpsnr"] <= PSNR_TOL, st


@pytest.mark.parametrize("pos", [(0, 1024 - 192), (400, 300)])
def test_c5_image31_tiles(c5_batch, oracle, pos):
    cfg, model, u, _ = c5_batch
    _, f31 = synth.noisy_image(cfg, 31)
    t, marg = 192, cfg.T * (cfg.m - 1)
    y, x = pos
    oy0, oy1 = max(0, y - marg), min(cfg.H, y + t + marg)
    ox0, ox1 = max(0, x - marg), min(cfg.W, x + t + marg)
    ref = oracle.run_diffusion(f31[oy0:oy1, ox0:ox1].astype(np.float64), model)
    ref = ref[y - oy0:y - oy0 + t, x - ox0:x - ox0 + t]
    st = parity_stats(u[31][y:y + t, x:x + t], ref)
    assert st["rel"] <= REL_TOL, st

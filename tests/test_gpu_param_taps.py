"""The large-tile CUDA-core kernels read the filter taps either from the
kernel parameter space (uniform datapath, the default) or from shared
memory (tnrd_set_param_taps(0)).  The arithmetic is the same FMA chain in
the same order, so the tile kernel must agree bit for bit; the split kernel
agrees bit for bit when both use the same filter groups (and to fp32
summation order otherwise).  Both variants meet the parity bar."""
import numpy as np
import pytest

from conftest import parity_stats

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

pytestmark = pytest.mark.gpu


def _despeckle(f, model, param_taps, mode):
    import torch
    _lib.set_param_taps(param_taps)
    _lib.set_stage_kernel(mode)
    try:
        dm = tn.device_model_for(model)
        u = dm.despeckle(torch.from_numpy(f).cuda())
        return u.cpu().numpy()
    finally:
        _lib.set_param_taps(True)
        _lib.set_stage_kernel(_lib.KERNEL_AUTO)


CASES = [  # (H, W, m, nk, T) -- nk odd / not a multiple of 4 exercises the zero-filter padding
    (512, 512, 7, 48, 2),
    (230, 301, 7, 7, 2),
    (130, 67, 5, 24, 2),
    (97, 200, 3, 10, 3),
    (150, 170, 9, 80, 2),
    (70, 90, 9, 5, 2),
]


@pytest.mark.parametrize("H,W,m,nk,T", CASES)
def test_tile_kernel_param_taps_bit_identical(cuda, H, W, m, nk, T):
    model = synth.make_model(m, nk, T, 63, seed=H + W + m)
    f = np.random.default_rng(H * W).uniform(0, 300, (H, W)).astype(np.float32)
    a = _despeckle(f, model, True, _lib.KERNEL_LARGE_TILES)
    b = _despeckle(f, model, False, _lib.KERNEL_LARGE_TILES)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("H,W,m,nk,T", CASES)
def test_split_kernel_param_taps(cuda, oracle, H, W, m, nk, T):
    model = synth.make_model(m, nk, T, 63, seed=H + W + m)
    f = np.random.default_rng(H * W).uniform(0, 300, (H, W)).astype(np.float32)
    a = _despeckle(f, model, True, _lib.KERNEL_SPLIT_LARGE)
    a2 = _despeckle(f, model, True, _lib.KERNEL_SPLIT_LARGE)
    b = _despeckle(f, model, False, _lib.KERNEL_SPLIT_LARGE)
    assert np.array_equal(a, a2)                      # bit-reproducible
    assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-5  # fp32 summation order at most
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    assert parity_stats(a, ref)["rel"] <= 1e-4


def test_c2_auto_param_taps_parity(cuda, oracle):
    cfg = synth.CONFIGS["c2"]
    clean, f = synth.noisy_image(cfg, 0)
    model = synth.config_model(cfg)
    u = _despeckle(f, model, True, _lib.KERNEL_AUTO)
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    st = parity_stats(u, ref, clean)
    assert st["rel"] <= 1e-4 and st["dpsnr"] <= 0.01, st

"""The large-tile CUDA-core kernels read the filter taps either from the
kernel parameter space (uniform datapath) with the cubic RBF table (the
default), or from shared memory with the degree-7 table
(tnrd_set_param_taps(0)).  The convolutions are the same FMA chains in the
same order; phi differs by the two interpolants (both at the fp32
resolution of phi), so the variants agree to ~1e-6 relative and both meet
the parity bar; each is bit-reproducible."""
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
def test_tile_kernel_param_taps(cuda, H, W, m, nk, T):
    model = synth.make_model(m, nk, T, 63, seed=H + W + m)
    f = np.random.default_rng(H * W).uniform(0, 300, (H, W)).astype(np.float32)
    a = _despeckle(f, model, True, _lib.KERNEL_LARGE_TILES)
    a2 = _despeckle(f, model, True, _lib.KERNEL_LARGE_TILES)
    b = _despeckle(f, model, False, _lib.KERNEL_LARGE_TILES)
    assert np.array_equal(a, a2)
    assert np.max(np.abs(a - b) / np.abs(b)) <= 2e-5


@pytest.mark.parametrize("H,W,m,nk,T", CASES)
def test_split_kernel_param_taps(cuda, oracle, H, W, m, nk, T):
    model = synth.make_model(m, nk, T, 63, seed=H + W + m)
    f = np.random.default_rng(H * W).uniform(0, 300, (H, W)).astype(np.float32)
    a = _despeckle(f, model, True, _lib.KERNEL_SPLIT_LARGE)
    a2 = _despeckle(f, model, True, _lib.KERNEL_SPLIT_LARGE)
    b = _despeckle(f, model, False, _lib.KERNEL_SPLIT_LARGE)
    assert np.array_equal(a, a2)                      # bit-reproducible
    assert np.max(np.abs(a - b) / np.abs(b)) <= 2e-5  # the two RBF interpolants
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


def test_models_beyond_the_parameter_block_fall_back(cuda, oracle):
    """m = 7 with 60 filters does not fit the 10 KB TapBlock: the large-tile
    launches fall back to the shared-memory-taps kernels (same results as
    forcing them) and still meet the parity bar."""
    model = synth.make_model(7, 60, 2, 63, seed=11)
    f = np.random.default_rng(5).uniform(0, 300, (200, 260)).astype(np.float32)
    for mode in (_lib.KERNEL_LARGE_TILES, _lib.KERNEL_SPLIT_LARGE):
        a = _despeckle(f, model, True, mode)
        b = _despeckle(f, model, False, mode)
        assert np.array_equal(a, b)
        ref = oracle.run_diffusion(f.astype(np.float64), model)
        assert parity_stats(a, ref)["rel"] <= 1e-4


@pytest.mark.parametrize("mode", [_lib.KERNEL_LARGE_TILES, _lib.KERNEL_SPLIT_LARGE], ids=["tile", "split"])
def test_padded_row_stride_matches_contiguous(cuda, mode):
    """Row stride ld > W and image stride > ld * H (views into wider, taller
    buffers) give the same bits as the dense layout."""
    torch = cuda
    model = synth.make_model(7, 10, 2, 63, seed=4)
    B, H, W = 2, 150, 181
    f = np.random.default_rng(9).uniform(0, 300, (B, H, W)).astype(np.float32)
    dm = tn.device_model_for(model)
    _lib.set_stage_kernel(mode)
    try:
        dense = dm.despeckle(torch.from_numpy(f).cuda())
        big = [torch.zeros(B, H + 5, W + 13, device="cuda") for _ in range(3)]
        fv, ov, wv = (b[:, :H, :W] for b in big)
        fv.copy_(torch.from_numpy(f).cuda())
        got = dm.despeckle(fv, out=ov, work=wv)
    finally:
        _lib.set_stage_kernel(_lib.KERNEL_AUTO)
    assert got.stride() == ov.stride() and got.stride(-2) == W + 13
    assert torch.equal(got.contiguous(), dense)

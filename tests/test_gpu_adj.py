"""Tensor-core adjoint stage (mode 12, csrc/tnrd_stage_adj.cuh): phi_kernel
(CUDA cores: z, phi = RBF(z) once per pixel, written in the GEMM's A layout
with the mirrored copies the reference's phi padding implies,
diffusion.py:178-180) + adj_kernel (tcgen05 3xTF32 GEMM psi = Phi K^T, shifted
sum in the epilogue, reaction).  Parity against the reference's golden vectors
and the oracle at the north_star bar (1e-4 relative, 0.01 dB)."""
import numpy as np
import pytest

from conftest import golden_model, golden_names, load_golden, parity_stats

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

pytestmark = pytest.mark.gpu
KERNEL_TC_ADJOINT = _lib.KERNEL_TC_ADJOINT


@pytest.fixture
def adjoint(cuda):
    _lib.set_stage_kernel(KERNEL_TC_ADJOINT)
    yield
    _lib.set_stage_kernel(_lib.KERNEL_AUTO)


def _m(name):
    return int(load_golden(name)["m"])


@pytest.mark.parametrize("name", [n for n in golden_names(full_only=True) if _m(n) in (5, 7)])
def test_golden_adjoint(adjoint, name):
    g = load_golden(name)
    u, _ = tn.run_diffusion(g["f"], golden_model(g))
    st = parity_stats(u, g["u"], g.get("clean"))
    tol = 5e-3 if name == "huge_weights" else 1e-4   # cubic-table tails, as in test_gpu_tiles.py
    assert st["rel"] <= tol and st["abs_degenerate"] <= 1e-9, st


@pytest.mark.parametrize("H,W,m,nk", [(97, 130, 7, 6), (7, 200, 7, 5), (200, 7, 7, 8), (64, 64, 7, 3),
                                      (130, 67, 5, 7), (128, 104, 7, 12), (150, 215, 7, 48), (3, 3, 7, 2)])
def test_shapes_adjoint(adjoint, oracle, H, W, m, nk):
    """Ragged / tiny shapes, column groups that end inside and at the image
    edge, odd filter counts (zero-padded chunks)."""
    model = synth.make_model(m, nk, 2, 63, seed=H * 1000 + W)
    f = np.random.default_rng(H + W).uniform(0, 300, (H, W)).astype(np.float32)
    u, _ = tn.run_diffusion(f, model)
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    assert parity_stats(u, ref)["rel"] <= 1e-4


def test_c2_full_adjoint_two_launches_per_stage(adjoint, oracle):
    cfg = synth.CONFIGS["c2"]
    clean, f = synth.noisy_image(cfg, 0)
    model = synth.config_model(cfg)
    _lib.launch_count_reset()
    u, _ = tn.run_diffusion(f, model)
    assert _lib.launch_count() == 2 * cfg.T
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    st = parity_stats(u, ref, clean)
    assert st["rel"] <= 1e-4 and st["dpsnr"] <= 0.01, st


def test_batch_bit_reproducible_adjoint(adjoint):
    import torch
    model = synth.make_model(7, 12, 3, 63, seed=11)
    dm = tn.device_model_for(model)
    rng = np.random.default_rng(4)
    fs = [rng.uniform(0, 300, (150, 170)).astype(np.float32) for _ in range(3)]
    fb = torch.from_numpy(np.stack(fs)).cuda()
    ub = dm.despeckle(fb)
    assert torch.equal(ub, dm.despeckle(fb))
    for i, fi in enumerate(fs):
        assert torch.equal(dm.despeckle(torch.from_numpy(fi).cuda()), ub[i])


def test_matches_cuda_core_kernels_adjoint(cuda):
    torch = cuda
    cfg = synth.CONFIGS["c3"]
    model = synth.config_model(cfg)
    f = torch.from_numpy(synth.noisy_batch(cfg, range(4))).cuda()
    dm = tn.device_model_for(model)
    a = dm.despeckle(f).cpu().numpy()
    _lib.set_stage_kernel(KERNEL_TC_ADJOINT)
    try:
        b = dm.despeckle(f).cpu().numpy()
    finally:
        _lib.set_stage_kernel(_lib.KERNEL_AUTO)
    assert np.max(np.abs(a - b) / a) < 2e-5


def test_error_contract_and_force_output_adjoint(adjoint, oracle):
    g = load_golden("overflow_stage1")
    with pytest.raises(FloatingPointError, match=str(g["raises"])):
        tn.run_diffusion(g["f"], golden_model(g))
    model = synth.make_model(7, 10, 2, 63, seed=5)
    f = np.full((40, 40), 5.0, np.float32)
    f[3, 7] = -1.0
    with pytest.raises(ValueError):
        tn.run_diffusion(f, model)
    stage = model.stages[0]
    rng = np.random.default_rng(9)
    f = rng.uniform(1, 255, (90, 110)).astype(np.float32).astype(np.float64)
    u0 = rng.uniform(1, 255, (90, 110)).astype(np.float32).astype(np.float64)
    u1, tr = tn.diffusion_step(u0, f, stage, model)
    kern = stage.kernels(model.basis, model.filter_size)
    gr = model.rbf
    force = oracle.force(u0, kern, stage.weights, gr.centers, gr.gamma)
    assert np.abs(tr.u_tilde - (u0 - force)).max() <= 1e-4 * np.abs(u0).max()
    ref = oracle.stage(u0, f, kern, stage.weights, gr.centers, gr.gamma, stage.lam)
    assert parity_stats(u1, ref)["rel"] <= 1e-4

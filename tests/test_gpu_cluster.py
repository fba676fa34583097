"""Cluster stage kernel (modes 10 / 11): ONE launch per stage on small grids
-- the CTAs of a thread-block cluster split a tile's filter groups and sum
their partial forces in rank order through distributed shared memory
(diffusion_step, reference diffusion.py:184-194, as one fused operator).
Parity against the reference's golden vectors and the oracle for every
cluster size, bit-reproducibility / position independence for a fixed size,
the strip mode, both reaction variants and the force output."""
import numpy as np
import pytest

from conftest import golden_model, golden_names, load_golden, parity_stats

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

pytestmark = pytest.mark.gpu

MODES = {"cluster_large": _lib.KERNEL_CLUSTER_LARGE, "cluster_small": _lib.KERNEL_CLUSTER_SMALL}


@pytest.fixture(params=list(MODES.values()), ids=list(MODES.keys()))
def cluster(cuda, request):
    _lib.set_stage_kernel(request.param)
    yield request.param
    _lib.set_cluster_size(0)
    _lib.set_stage_kernel(_lib.KERNEL_AUTO)


@pytest.mark.parametrize("name", golden_names(full_only=True))
def test_golden_cluster(cluster, name):
    g = load_golden(name)
    u, _ = tn.run_diffusion(g["f"], golden_model(g))
    st = parity_stats(u, g["u"], g.get("clean"))
    tol = 1e-4
    if name == "huge_weights" and cluster == _lib.KERNEL_CLUSTER_LARGE:
        # the cubic table's tail-relative error, as in test_gpu_tiles.py
        assert np.all(np.isfinite(u))
        tol = 5e-3
    assert st["rel"] <= tol and st["abs_degenerate"] <= 1e-9, st


@pytest.mark.parametrize("cl", [2, 3, 4, 5, 8])
def test_every_cluster_size_meets_the_oracle(cluster, oracle, cl):
    """Group ranges that divide evenly, unevenly (6 groups on 4 / 5 CTAs) and
    clusters with more CTAs than groups (idle ranks contribute zeros)."""
    _lib.set_cluster_size(cl)
    for m, nk, seed in ((7, 12, 1), (5, 24, 2), (7, 3, 3)):
        model = synth.make_model(m, nk, 2, 63, seed=seed)
        f = np.random.default_rng(seed).uniform(0, 300, (150, 131)).astype(np.float32)
        u, _ = tn.run_diffusion(f, model)
        ref = oracle.run_diffusion(f.astype(np.float64), model)
        assert parity_stats(u, ref)["rel"] <= 1e-4, (cl, m, nk)


@pytest.mark.parametrize("H,W,m", [(3, 200, 7), (200, 3, 7), (97, 130, 9), (130, 67, 5), (64, 64, 3), (4, 4, 7)])
def test_edge_shapes_cluster(cluster, oracle, H, W, m):
    model = synth.make_model(m, 6, 2, 63, seed=H * 1000 + W)
    f = np.random.default_rng(H + W).uniform(0, 300, (H, W)).astype(np.float32)
    u, _ = tn.run_diffusion(f, model)
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    assert parity_stats(u, ref)["rel"] <= 1e-4


def test_c1_c2_full_cluster_one_launch_per_stage(cluster, oracle):
    for name in ("c1", "c2"):
        cfg = synth.CONFIGS[name]
        clean, f = synth.noisy_image(cfg, 0)
        model = synth.config_model(cfg)
        _lib.launch_count_reset()
        u, _ = tn.run_diffusion(f, model)
        assert _lib.launch_count() == cfg.T          # one fused launch per stage
        ref = oracle.run_diffusion(f.astype(np.float64), model)
        st = parity_stats(u, ref, clean)
        assert st["rel"] <= 1e-4 and st["dpsnr"] <= 0.01, (name, st)


def test_projected_variant_and_force_output_cluster(cluster, oracle):
    model = synth.make_model(7, 10, 2, 63, seed=5)
    stage = model.stages[0]
    rng = np.random.default_rng(9)
    f = rng.uniform(1, 255, (90, 110)).astype(np.float32).astype(np.float64)
    u0 = rng.uniform(1, 255, (90, 110)).astype(np.float32).astype(np.float64)
    u1, tr = tn.diffusion_step(u0, f, stage, model)   # u_next and the force from one launch
    kern = stage.kernels(model.basis, model.filter_size)
    g = model.rbf
    force = oracle.force(u0, kern, stage.weights, g.centers, g.gamma)
    assert np.abs(tr.u_tilde - (u0 - force)).max() <= 1e-4 * np.abs(u0).max()
    ref = oracle.stage(u0, f, kern, stage.weights, g.centers, g.gamma, stage.lam)
    assert parity_stats(u1, ref)["rel"] <= 1e-4
    g = load_golden("projected_m7")
    u, _ = tn.run_diffusion(g["f"], golden_model(g))
    assert parity_stats(u, g["u"])["rel"] <= 1e-4


def test_strips_bit_identical_cluster(cluster):
    """Row strips (TOP / BOTTOM halo modes) give the whole image's bits when
    the cluster size is the same for both."""
    import torch
    from test_gpu_strips import lockstep_strips
    _lib.set_cluster_size(4)
    model = synth.make_model(7, 8, 3, 63, seed=3)
    H, W = 230, 140
    f = torch.from_numpy(np.random.default_rng(2).uniform(0, 300, (H, W)).astype(np.float32)).cuda()
    dm = tn.device_model_for(model)
    whole = dm.despeckle(f)
    assert torch.equal(lockstep_strips(dm, f, 3, model.num_stages), whole)


@pytest.mark.parametrize("cl", [0, 4])
def test_cluster_reproducible_and_position_independent(cluster, cl):
    """Rank-ordered summation: repeated runs are bit-identical; with a fixed
    cluster size a batch equals its images one by one."""
    import torch
    _lib.set_cluster_size(cl)
    model = synth.make_model(7, 12, 3, 63, seed=11)
    dm = tn.device_model_for(model)
    rng = np.random.default_rng(4)
    fs = [rng.uniform(0, 300, (150, 170)).astype(np.float32) for _ in range(3)]
    fb = torch.from_numpy(np.stack(fs)).cuda()
    ub = dm.despeckle(fb)
    assert torch.equal(ub, dm.despeckle(fb))
    if cl:
        for i, fi in enumerate(fs):
            assert torch.equal(dm.despeckle(torch.from_numpy(fi).cuda()), ub[i])


def test_cluster_matches_tile_kernel_to_summation_order(cuda):
    torch = cuda
    cfg = synth.CONFIGS["c2"]
    model = synth.config_model(cfg)
    f = torch.from_numpy(synth.noisy_image(cfg, 0)[1]).cuda()
    dm = tn.device_model_for(model)
    try:
        _lib.set_stage_kernel(_lib.KERNEL_CLUSTER_LARGE)
        a = dm.despeckle(f).cpu().numpy()
        _lib.set_stage_kernel(_lib.KERNEL_LARGE_TILES)
        b = dm.despeckle(f).cpu().numpy()
    finally:
        _lib.set_stage_kernel(_lib.KERNEL_AUTO)
    assert np.max(np.abs(a - b) / b) < 1e-5


def test_error_contract_cluster(cluster):
    """Non-finite stage index and input validation through the cluster path."""
    g = load_golden("overflow_stage1")
    with pytest.raises(FloatingPointError, match=str(g["raises"])):
        tn.run_diffusion(g["f"], golden_model(g))
    model = synth.make_model(7, 4, 2, 63, seed=1)
    f = np.full((40, 40), 5.0, np.float32)
    f[3, 7] = -1.0
    with pytest.raises(ValueError):
        tn.run_diffusion(f, model)

"""GPU parity: the fused sm_100a path (through the C ABI) against the CPU
oracle and the reference's golden vectors.  Bar (BASELINE.json north_star):
max relative error <= 1e-4 on output pixels and |dPSNR| <= 0.01 dB."""
import numpy as np
import pytest

from conftest import golden_model, golden_names, load_golden, parity_stats

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import synth

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4      # north_star: max relative error on output pixels
PSNR_TOL = 0.01     # north_star: |dPSNR| in dB
DEG_ABS_TOL = 1e-9  # pixels whose reference value is < 1e-6 (f == 0)


@pytest.mark.parametrize("name", golden_names(full_only=True))
def test_golden_cases(cuda, name):
    g = load_golden(name)
    model = golden_model(g)
    u, traces = tn.run_diffusion(g["f"], model)
    assert traces is None
    st = parity_stats(u, g["u"], g.get("clean"))
    assert st["rel"] <= REL_TOL, st
    assert st["abs_degenerate"] <= DEG_ABS_TOL, st
    if "dpsnr" in st:
        assert st["dpsnr"] <= PSNR_TOL, st


@pytest.mark.parametrize("key", ["c1", "c2"])
def test_full_config_vs_oracle_and_golden(cuda, oracle, key):
    cfg = synth.CONFIGS[key]
    g = load_golden(f"{key}_full")
    clean, f = synth.noisy_image(cfg, 0)
    assert float(f.astype(np.float64).sum()) == float(g["f_sum"])
    model = synth.config_model(cfg)
    u, _ = tn.run_diffusion(f, model)
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    st = parity_stats(u, ref, clean)
    assert st["rel"] <= REL_TOL and st["dpsnr"] <= PSNR_TOL, st
    # and directly against the reference's own output crops / PSNR
    c = 24
    H, W = u.shape
    for k, v in dict(crop_tl=u[:c, :c], crop_br=u[H - c:, W - c:],
                     crop_c=u[H // 2 - c // 2:H // 2 + c // 2,
                              W // 2 - c // 2:W // 2 + c // 2]).items():
        assert np.max(np.abs(v - g[k]) / g[k]) <= REL_TOL, k
    assert abs(oracle.psnr(u, clean, 255.0) - float(g["psnr"])) <= PSNR_TOL


def test_c3_batch_subset(cuda, oracle):
    """Batched device entry on 8 images of C3 (2 per looks value, first and
    last index included) against the oracle, image by image."""
    torch = cuda
    cfg = synth.CONFIGS["c3"]
    model = synth.config_model(cfg)
    idx = [0, 1, 2, 3, 4, 5, 254, 255]
    pairs = [synth.noisy_image(cfg, i) for i in idx]
    f = torch.from_numpy(np.stack([p[1] for p in pairs])).cuda()
    u = tn.run_diffusion_batch(f, model).cpu().numpy()
    for j, (clean, fi) in enumerate(pairs):
        ref = oracle.run_diffusion(fi.astype(np.float64), model)
        st = parity_stats(u[j], ref, clean)
        assert st["rel"] <= REL_TOL and st["dpsnr"] <= PSNR_TOL, (idx[j], st)


@pytest.mark.parametrize("where", ["tl", "br", "top_mid", "interior",
                                   "strip_8192", "strip_4096", "strip_2048"])
def test_c4_tiles_with_margin(cuda, oracle, where):
    """C4 (16384^2): the despeckled scene restricted to a tile equals the
    oracle run on the tile plus a T*(m-1) = 30 px margin (the dependency
    radius after T stages).  The GPU runs on a band of the
    scene around the tile (64 px margin), mirrored only at true edges."""
    cfg = synth.CONFIGS["c4"]
    model = synth.config_model(cfg)
    N = cfg.H
    t = 96
    pos = {"tl": (0, 0), "br": (N - t, N - t), "top_mid": (0, N // 2 - t // 2),
           "interior": (5000, 9000), "strip_8192": (8192 - t // 2, 3000),
           "strip_4096": (4096 - t // 2, 16000), "strip_2048": (2048 - t // 2, 200)}[where]
    y, x = pos
    marg = cfg.T * (cfg.m - 1)
    # oracle on tile + margin (clipped at true image edges, where the mirror applies)
    oy0, oy1 = max(0, y - marg), min(N, y + t + marg)
    ox0, ox1 = max(0, x - marg), min(N, x + t + marg)
    fo = synth.scene_crop(cfg, oy0, oy1, ox0, ox1).astype(np.float64)
    ref = oracle.run_diffusion(fo, model)[y - oy0:y - oy0 + t, x - ox0:x - ox0 + t]
    # GPU on a wider crop (same rule, bigger margin) -> identical interior
    gm = 2 * marg + 4
    gy0, gy1 = max(0, y - gm), min(N, y + t + gm)
    gx0, gx1 = max(0, x - gm), min(N, x + t + gm)
    fg = synth.scene_crop(cfg, gy0, gy1, gx0, gx1)
    u, _ = tn.run_diffusion(fg, model)
    u = u[y - gy0:y - gy0 + t, x - gx0:x - gx0 + t]
    st = parity_stats(u, ref)
    assert st["rel"] <= REL_TOL, st


@pytest.mark.slow
def test_c5_tile_with_margin(cuda, oracle):
    """C5 (9x9, Nk=80, T=8): a 192^2 corner tile of image 0 vs the oracle on
    tile + 64 px margin (T*(m-1))."""
    cfg = synth.CONFIGS["c5"]
    model = synth.config_model(cfg)
    clean, f = synth.noisy_image(cfg, 0)
    u, _ = tn.run_diffusion(f, model)
    t, marg = 192, cfg.T * (cfg.m - 1)
    for (y, x) in [(0, 0), (cfg.H - t, cfg.W // 2)]:
        oy0, oy1 = max(0, y - marg), min(cfg.H, y + t + marg)
        ox0, ox1 = max(0, x - marg), min(cfg.W, x + t + marg)
        ref = oracle.run_diffusion(f[oy0:oy1, ox0:ox1].astype(np.float64), model)
        ref = ref[y - oy0:y - oy0 + t, x - ox0:x - ox0 + t]
        st = parity_stats(u[y:y + t, x:x + t], ref)
        assert st["rel"] <= REL_TOL, st


def test_c5_batch_matches_single(cuda):
    """Batch launch over images == per-image launches: bit-exact once the
    cluster size is pinned (auto picks it from the grid size, and the
    partial forces are summed in cluster-rank order), equal to fp32
    summation order otherwise."""
    from paper_1702_07482_b200 import _lib
    torch = cuda
    cfg = synth.CONFIGS["c5"]
    model = synth.config_model(cfg)
    fs = [synth.noisy_image(cfg, i, 256, 256)[1] for i in range(3)]
    fb = torch.from_numpy(np.stack(fs)).cuda()
    auto = tn.run_diffusion_batch(fb, model).cpu().numpy()
    for i, fi in enumerate(fs):
        ui = tn.run_diffusion_batch(torch.from_numpy(fi).cuda(), model).cpu().numpy()
        assert np.max(np.abs(auto[i] - ui) / ui) < 1e-5
    _lib.set_cluster_size(4)
    try:
        ub = tn.run_diffusion_batch(fb, model).cpu().numpy()
        for i, fi in enumerate(fs):
            ui = tn.run_diffusion_batch(torch.from_numpy(fi).cuda(), model).cpu().numpy()
            np.testing.assert_array_equal(ub[i], ui)
    finally:
        _lib.set_cluster_size(0)


@pytest.mark.parametrize("H,W,m", [(1, 1, 1), (3, 200, 7), (200, 3, 7), (5, 5, 9),
                                   (33, 65, 3), (64, 31, 5), (97, 130, 9)])
def test_edge_shapes(cuda, oracle, H, W, m):
    """Ragged / tiny shapes, including m close to 2*min(H, W)+1."""
    if m > 2 * min(H, W) + 1 or m == 1:
        pytest.skip("degenerate")
    model = synth.make_model(m, 6, 2, 63, seed=H * 1000 + W)
    f = np.random.default_rng(H + W).uniform(0, 300, (H, W)).astype(np.float32)
    u, _ = tn.run_diffusion(f, model)
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    st = parity_stats(u, ref)
    assert st["rel"] <= REL_TOL, st


@pytest.mark.parametrize("key", ["c1", "c2", "c5"])
def test_rbf_polynomial_tables_accuracy(cuda, key):
    """The per-interval degree-11 fits of every phi_i are exact to far below
    fp32 resolution (checked in float64 at model creation)."""
    dm = tn.device_model_for(synth.config_model(synth.CONFIGS[key]))
    err, err32, scale, ni = dm.rbf_fit
    assert dm.fast_rbf and ni > 0
    assert err <= 1e-9 * scale, dm.rbf_fit      # interpolation itself
    assert err32 <= 1e-7 * scale, dm.rbf_fit    # ~ fp32 resolution of phi


@pytest.mark.parametrize("key", ["c1", "c2", "c5"])
def test_rbf_cubic_tables_accuracy(cuda, key):
    """The cubic tables of the parameter-space-taps kernels (10 intervals
    per centre spacing) interpolate phi_i to the fp32 resolution of phi:
    below 2e-7 of sum|w| with float64 and with fp32 coefficients."""
    dm = tn.device_model_for(synth.config_model(synth.CONFIGS[key]))
    err, err32, ni = dm.rbf_fit_cubic
    scale = dm.rbf_fit[2]
    assert ni > 0
    assert err <= 2e-7 * scale, dm.rbf_fit_cubic
    assert err32 <= 2e-7 * scale, dm.rbf_fit_cubic


def test_direct_rbf_path_parity(cuda, oracle):
    """A bandwidth so narrow that the polynomial table would not fit in
    shared memory selects the direct all-centre RBF path."""
    model = synth.make_model(7, 8, 2, 63, seed=3)
    model.rbf = tn.RbfGrid(63, 310.0, bandwidth=1.5)
    dm = tn.device_model_for(model)
    assert not dm.fast_rbf
    f = np.random.default_rng(5).uniform(1, 255, (70, 90)).astype(np.float32)
    u, _ = tn.run_diffusion(f, model)
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    assert parity_stats(u, ref)["rel"] <= REL_TOL

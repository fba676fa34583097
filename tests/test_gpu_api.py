"""The reference's hot-path unit tests, restated against the GPU drop-in.

Mirrors /root/reference/pkg/tests/test_diffusion.py, test_imageops.py,
test_speckle.py and test_acceptance.py gates 1 and 4, with tolerances
widened from float64 round-off to the fp32 parity bar where the GPU
computes in fp32."""
import math

import numpy as np
import pytest

from conftest import load_golden

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

pytestmark = pytest.mark.gpu


def make_model(rng, m=3, nk=2, T=1, M=7, beta=0.0, weight_scale=0.05):
    # reference tests/test_diffusion.py:12-22
    grid = tn.RbfGrid(count=M, radius=310.0)
    stages = []
    for _ in range(T):
        c = rng.standard_normal((nk, m * m - 1))
        c /= np.linalg.norm(c, axis=1, keepdims=True)
        w = weight_scale * rng.standard_normal((nk, M))
        stages.append(tn.StageParams(beta=beta, coeffs=c, weights=w))
    return tn.DiffusionModel(stages=stages, filter_size=m, looks=4, rbf=grid)


def zero_weight_model(rng, beta, T=1):
    model = make_model(rng, T=T, beta=beta)
    for s in model.stages:
        s.weights[:] = 0.0
    return model


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


# ------------------------------------------------------------- diffusion_step

def test_zero_weights_reduces_to_prox(cuda, oracle):
    rng = np.random.default_rng(2)
    model = zero_weight_model(rng, beta=0.5)
    f = rng.uniform(1, 10, (12, 12)).astype(np.float32).astype(np.float64)
    u = rng.uniform(1, 10, (12, 12)).astype(np.float32).astype(np.float64)
    out, trace = tn.diffusion_step(u, f, model.stages[0], model)
    np.testing.assert_array_equal(trace.u_tilde, u)  # force is exactly 0
    assert rel(out, oracle.prox_idiv(u, f, math.exp(0.5))) < 1e-6


def test_zero_weights_tiny_lambda_is_identity(cuda):
    rng = np.random.default_rng(3)
    model = zero_weight_model(rng, beta=-40.0)
    f = rng.uniform(1, 10, (12, 12))
    u = rng.uniform(1, 10, (12, 12)).astype(np.float32).astype(np.float64)
    out, _ = tn.diffusion_step(u, f, model.stages[0], model)
    assert np.abs(out - u).max() < 1e-5


def test_compositional_oracle(cuda, oracle):
    rng = np.random.default_rng(4)
    model = make_model(rng, nk=3, M=9)
    stage = model.stages[0]
    f = rng.uniform(1, 200, (16, 16)).astype(np.float32).astype(np.float64)
    u = rng.uniform(1, 200, (16, 16)).astype(np.float32).astype(np.float64)
    out, trace = tn.diffusion_step(u, f, stage, model)
    kern = stage.kernels(model.basis, model.filter_size)
    g = model.rbf
    expected = oracle.stage(u, f, kern, stage.weights, g.centers, g.gamma, stage.lam)
    assert rel(out, expected) < 1e-5
    force = oracle.force(u, kern, stage.weights, g.centers, g.gamma)
    assert np.abs(trace.u_tilde - (u - force)).max() < 1e-4 * np.abs(u).max()
    # diffusion_force with explicit kernels
    fgpu, z, phi, design = tn.diffusion_force(u, stage, kern, model.rbf)
    assert z is None and phi is None and design is None
    assert np.abs(fgpu - force).max() < 1e-4 * max(1.0, np.abs(force).max())


def test_constant_image_closed_form(cuda):
    rng = np.random.default_rng(5)
    lam = math.exp(0.3)
    model = zero_weight_model(rng, beta=0.3)
    c = 4.0
    out, _ = tn.run_diffusion(np.full((8, 8), c), model)
    expected = (c + math.sqrt(c * c + 8 * (1 + 2 * lam) * lam * c * c)) / (2 * (1 + 2 * lam))
    assert np.abs(out - expected).max() < 1e-5 * expected


def test_positivity_and_determinism(cuda):
    # reference test_diffusion.py:129-137 and acceptance gate 4 (:125-139)
    rng = np.random.default_rng(404)
    for trial in range(100):
        T = int(rng.integers(1, 4))
        nk = int(rng.integers(1, 5))
        model = make_model(rng, m=3, nk=nk, T=T, M=7, beta=float(rng.normal(0.0, 0.5)))
        side = int(rng.integers(8, 17))
        f = rng.uniform(0.0, 255.0, (side, side))
        out1, _ = tn.run_diffusion(f, model)
        out2, _ = tn.run_diffusion(f, model)
        assert np.all(out1 > 0.0)
        np.testing.assert_array_equal(out1, out2)


def test_prefix_invariance(cuda):
    # reference test_diffusion.py:139-148, through the stage API
    rng = np.random.default_rng(7)
    model = make_model(rng, T=3)
    f = rng.uniform(1, 255, (10, 10))
    u0 = np.maximum(f, 1e-6)
    u1, _ = tn.diffusion_step(u0, f, model.stages[0], model)
    model.stages[2].weights += 0.1
    model.stages[2].beta += 0.5
    u1b, _ = tn.diffusion_step(u0, f, model.stages[0], model)
    np.testing.assert_array_equal(u1, u1b)


def test_in_place_param_edit_invalidates_device_cache(cuda):
    rng = np.random.default_rng(8)
    model = make_model(rng, T=2)
    f = rng.uniform(1, 255, (10, 10))
    a, _ = tn.run_diffusion(f, model)
    model.stages[1].weights *= 3.0
    b, _ = tn.run_diffusion(f, model)
    assert not np.array_equal(a, b)


# ------------------------------------------------------------- error contract

def test_errors_match_reference(cuda):
    rng = np.random.default_rng(9)
    model = make_model(rng, m=7, nk=2)
    with pytest.raises(ValueError, match="nonnegative"):
        tn.run_diffusion(-np.ones((10, 10)), model)
    bad = np.ones((10, 10))
    bad[3, 3] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        tn.run_diffusion(bad, model)
    with pytest.raises(ValueError, match="2D"):
        tn.run_diffusion(np.ones(10), model)
    with pytest.raises(ValueError, match="degenerate"):
        tn.run_diffusion(np.ones((2, 2)), model)
    with pytest.raises(NotImplementedError):
        tn.run_diffusion(np.ones((10, 10)), model, keep_traces=True)


def test_nonfinite_stage_matches_reference(cuda):
    """The reference raises only when its float64 image is non-finite
    (diffusion.py:238-239).  Stage 1 weights of 1e301 overflow its u~^2 in
    stage 1 (golden 'overflow_stage1', written by the reference): the GPU
    raises with the same message and stage index."""
    from conftest import golden_model
    g = load_golden("overflow_stage1")
    with pytest.raises(FloatingPointError, match=str(g["raises"])):
        tn.run_diffusion(g["f"], golden_model(g))
    # device entry: same stage through the status block
    with pytest.raises(FloatingPointError, match="after stage 1"):
        tn.run_diffusion_batch(cuda.from_numpy(g["f"].astype(np.float32)).cuda(), golden_model(g))


def test_huge_weights_finish_like_reference(cuda):
    """Weights of 1e30 drive |u~| to ~1e31, whose fp32 square overflows;
    the reference (float64) finishes with a finite image (max ~1.4e29) and
    so must the GPU (prox evaluated with an exact power-of-two rescale,
    tnrd_stage.cuh prox_idiv_f).  Parity at the north_star bar."""
    from conftest import golden_model
    g = load_golden("huge_weights")
    u, _ = tn.run_diffusion(g["f"], golden_model(g))
    assert np.all(np.isfinite(u))
    assert np.max(np.abs(u - g["u"]) / np.abs(g["u"])) <= 1e-4


def test_prox_large_values_match_reference(cuda):
    """tnrd_prox_idiv at |u~| up to 1e37, f up to 1e19 (golden 'prox_large'
    from the reference): finite wherever the reference is; relative error
    <= 1e-6 where u~ >= 0.  For u~ < 0 the reference's naive float64 formula
    cancels (speckle.py:119-121), so those entries are checked against the
    stable float64 form 4 lam f^2 / (sqrt(u~^2 + 8 a lam f^2) - u~)."""
    g = load_golden("prox_large")
    ut, f = g["u_tilde"], g["f"]
    for i, lam in enumerate(g["lams"]):
        o = tn.prox_idiv(ut, f, float(lam))
        assert np.all(np.isfinite(o))
        pos = ut >= 0
        assert np.max(np.abs(o[pos] - g[f"out_{i}"][pos]) / g[f"out_{i}"][pos]) <= 1e-6
        a = 1.0 + 2.0 * lam
        ff = np.maximum(f, 1e-6)
        stable = 4 * lam * ff ** 2 / (np.sqrt(ut ** 2 + 8 * a * lam * ff ** 2) - ut)
        neg = (ut < 0) & (stable > 1e-30)
        assert np.max(np.abs(o[neg] - stable[neg]) / stable[neg]) <= 1e-5


def test_device_entry_validates_f(cuda):
    torch = cuda
    model = synth.make_model(5, 4, 2, 63, seed=2)
    f = torch.rand(2, 20, 20, device="cuda") * 100
    f[1, 5, 5] = -1.0
    with pytest.raises(ValueError, match="nonnegative"):
        tn.run_diffusion_batch(f, model)
    f[1, 5, 5] = float("inf")
    with pytest.raises(ValueError, match="non-finite"):
        tn.run_diffusion_batch(f, model)


# ------------------------------------------------------------- primitives

def _mirror(j, n):
    return -1 - j if j < 0 else (2 * n - 1 - j if j >= n else j)


def test_conv2d_bruteforce_and_golden(cuda):
    from conftest import load_golden
    rng = np.random.default_rng(2)
    img = rng.normal(size=(16, 16))
    k = rng.normal(size=(5, 5))
    ref = np.zeros_like(img)
    for i in range(16):
        for j in range(16):
            ref[i, j] = sum(k[2 + p, 2 + q] * img[_mirror(i - p, 16), _mirror(j - q, 16)]
                            for p in range(-2, 3) for q in range(-2, 3))
    assert np.abs(tn.conv2d(img, k) - ref).max() < 1e-5
    g = load_golden("conv2d")
    for m in (3, 5, 7, 9):
        out = tn.conv2d(g["img"], g[f"k{m}"])
        assert np.abs(out - g[f"out{m}"]).max() < 1e-5 * np.abs(g[f"out{m}"]).max()
    delta = np.zeros((5, 5))
    delta[2, 2] = 1.0
    img = rng.normal(size=(9, 13)).astype(np.float32).astype(np.float64)
    np.testing.assert_array_equal(tn.conv2d(img, delta), img)
    with pytest.raises(ValueError):
        tn.conv2d(np.zeros((4, 4)), np.zeros((11, 11)))
    with pytest.raises(ValueError):
        tn.conv2d(np.zeros((4, 4)), np.zeros((4, 4)))


def golden_section_prox(u_tilde, f, lam, tol=1e-9):
    def obj(u):
        return 0.5 * (u - u_tilde) ** 2 + lam * (u * u - 2 * f * f * math.log(u))
    a, b = 1e-12, abs(u_tilde) + 3.0 * f + 10.0
    phi = (math.sqrt(5.0) - 1.0) / 2.0
    c, d = b - phi * (b - a), a + phi * (b - a)
    fc, fd = obj(c), obj(d)
    while b - a > tol:
        if fc < fd:
            b, d, fd = d, c, fc
            c = b - phi * (b - a)
            fc = obj(c)
        else:
            a, c, fc = c, d, fd
            d = a + phi * (b - a)
            fd = obj(d)
    return 0.5 * (a + b)


def test_prox_known_value_minimizer_and_golden(cuda):
    from conftest import load_golden
    out = tn.prox_idiv(np.array([[2.0]]), np.array([[3.0]]), 1.0)
    assert abs(out[0, 0] - (2.0 + math.sqrt(220.0)) / 6.0) < 1e-6
    rng = np.random.default_rng(5)
    ut = rng.uniform(-10, 10, (100, 100))
    f = rng.uniform(1e-6, 10, (100, 100))
    for lam in (0.01, 1.0, 10.0):
        assert np.all(tn.prox_idiv(ut, f, lam) > 0)
    for _ in range(200):
        u_, f_, l_ = rng.uniform(-10, 10), rng.uniform(1e-3, 10), rng.uniform(1e-3, 10)
        closed = tn.prox_idiv(np.array([[u_]]), np.array([[f_]]), l_)[0, 0]
        assert abs(closed - golden_section_prox(u_, f_, l_)) < 1e-5 * max(1.0, closed)
    g = load_golden("prox")
    for i, lam in enumerate(g["lams"]):
        o = tn.prox_idiv(g["u_tilde"], g["f"], float(lam))
        assert np.max(np.abs(o - g[f"out_{i}"]) / g[f"out_{i}"]) < 1e-5
    with pytest.raises(ValueError):
        tn.prox_idiv(np.ones((2, 2)), np.ones((2, 2)), 0.0)


def test_launch_counter_counts_stages(cuda):
    """One launch per stage: the tile kernel, and the cluster kernel that
    auto picks on small grids; two (units + ordered reduction) for the split
    kernel (opt-in)."""
    model = synth.make_model(7, 8, 4, 63, seed=9)
    f = np.random.default_rng(0).uniform(1, 255, (40, 40))
    _lib.launch_count_reset()
    tn.run_diffusion(f, model)
    assert _lib.launch_count() == 4
    for mode, want in ((_lib.KERNEL_LARGE_TILES, 4), (_lib.KERNEL_SPLIT_SMALL, 8)):
        _lib.set_stage_kernel(mode)
        try:
            _lib.launch_count_reset()
            tn.run_diffusion(f, model)
            assert _lib.launch_count() == want
        finally:
            _lib.set_stage_kernel(_lib.KERNEL_AUTO)


def test_plan_graph_replay_matches_eager(cuda):
    """Plans replay a captured CUDA graph from the second call on: results
    must be bit-identical to the eager first call, errors still reported,
    and each call still counts its T cluster-kernel launches."""
    model = synth.make_model(7, 8, 4, 63, seed=21)
    f = np.random.default_rng(4).uniform(1, 255, (37, 45))
    outs = []
    for _ in range(4):
        _lib.launch_count_reset()
        u, _ = tn.run_diffusion(f, model)
        assert _lib.launch_count() == 4
        outs.append(u)
    for u in outs[1:]:
        np.testing.assert_array_equal(u, outs[0])
    bad = f.copy()
    bad[3, 4] = -1.0
    dm = tn.device_model_for(model)
    with pytest.raises(ValueError, match="nonnegative"):
        dm.despeckle_host(bad.astype(np.float32))   # graph path, device-side check
    np.testing.assert_array_equal(tn.run_diffusion(f, model)[0], outs[0])


# ------------------------------------------------------------- projected variant
# reference tests/test_diffusion.py:161-204

def test_projected_floor_respected(cuda):
    rng = np.random.default_rng(9)
    model = make_model(rng, T=3, weight_scale=0.2)
    model.variant = "projected"
    f = rng.uniform(0, 255, (16, 16))
    out, _ = tn.run_diffusion(f, model)
    assert np.all(out >= model.floor - 1e-6)


def test_projected_step_matches_primitives(cuda, oracle):
    rng = np.random.default_rng(11)
    model = make_model(rng, nk=2, M=7)
    model.variant = "projected"
    stage = model.stages[0]
    f = rng.uniform(1, 200, (10, 10)).astype(np.float32).astype(np.float64)
    u = rng.uniform(2, 200, (10, 10)).astype(np.float32).astype(np.float64)
    out, trace = tn.diffusion_step_projected(u, f, stage, model)
    kern = stage.kernels(model.basis, model.filter_size)
    g = model.rbf
    force = oracle.force(u, kern, stage.weights, g.centers, g.gamma)
    u_tilde = u - force - stage.lam * (1.0 / u - f ** 2 / u ** 3)
    expected = tn.smooth_max(u_tilde, model.floor)
    assert rel(out, expected) < 1e-5
    assert np.abs(trace.u_tilde - u_tilde).max() < 1e-4 * np.abs(u_tilde).max()


def test_projected_invalid_floor_and_smooth_max(cuda):
    rng = np.random.default_rng(10)
    with pytest.raises(ValueError, match="floor"):
        tn.DiffusionModel(stages=make_model(rng).stages, filter_size=3, looks=4,
                          variant="projected", floor=0.0)
    c = 1.0
    x = np.array([c + 10.0, c + 50.0])
    assert np.abs(tn.smooth_max(x, c) - x).max() < 1e-6
    x = np.array([c - 10.0, -50.0])
    assert np.abs(tn.smooth_max(x, c) - c).max() < 1e-6


def test_c_example_runs(cuda, tmp_path):
    """The plain-C client of the C ABI (examples/despeckle_c.c) builds and
    despeckles on the GPU (random model: only finiteness is checked)."""
    import os
    import re
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(repo, "paper_1702_07482_b200")
    exe = str(tmp_path / "despeckle_c")
    r = subprocess.run(["gcc", "-O2", "-I", os.path.join(repo, "include"),
                        os.path.join(repo, "examples", "despeckle_c.c"), "-L", lib, "-ltnrd",
                        f"-Wl,-rpath,{lib}", "-lm", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, "256", "320"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    m = re.search(r"checksum ([0-9.e+-]+);", r.stdout)
    assert m and np.isfinite(float(m.group(1))) and float(m.group(1)) > 0, r.stdout


def test_plan_despeckle_host_many_matches_single_calls(cuda):
    """tnrd_plan_despeckle_host_many (a stream of host images, copies
    overlapped with the next images' stages on chained twin plans) gives exactly the
    per-image results, and reports a bad image."""
    torch = cuda
    model = synth.make_model(7, 8, 3, 63, seed=31)
    dm = tn.device_model_for(model)
    rng = np.random.default_rng(8)
    fs = rng.uniform(1, 255, (5, 70, 90)).astype(np.float32)
    pinned = torch.from_numpy(fs).pin_memory()
    out = dm.despeckle_host_many(pinned.numpy())
    for i in range(5):
        np.testing.assert_array_equal(out[i], dm.despeckle_host(fs[i]))
    bad = fs.copy()
    bad[2, 5, 5] = -1.0
    with pytest.raises(ValueError, match="nonnegative"):
        dm.despeckle_host_many(bad)
    np.testing.assert_array_equal(dm.despeckle_host_many(fs), out)   # plan still usable

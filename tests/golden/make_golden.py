"""Generate golden vectors by running the REAL reference (specklediff) here.

Usage (in the build container, where /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed
as small .npz fixtures next to this script.  Each fixture holds the inputs
(f as fp32-exact float64, model parameters) and the reference output, full
for small cases and as border/centre crops plus global sums for the
full-size BASELINE configs C1 and C2.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import specklediff as sd  # noqa: E402  (the reference)
from specklediff.diffusion import DiffusionModel, StageParams  # noqa: E402
from specklediff.influence import RbfGrid  # noqa: E402

from paper_1702_07482_b200 import synth  # noqa: E402

CROP = 24


def ref_model(m, nk, T, M, seed, weight_scale=0.1, beta=0.0, radius=310.0,
              bandwidth=None, betas=None, variant="prox", floor=1.0):
    rng = np.random.default_rng(seed)
    stages = []
    for t in range(T):
        c = rng.standard_normal((nk, m * m - 1))
        c /= np.linalg.norm(c, axis=1, keepdims=True)
        w = weight_scale * rng.standard_normal((nk, M))
        b = beta if betas is None else betas[t]
        stages.append(StageParams(beta=b, coeffs=c, weights=w))
    grid = RbfGrid(count=M, radius=radius, bandwidth=bandwidth)
    return DiffusionModel(stages=stages, filter_size=m, looks=1, rbf=grid,
                          variant=variant, floor=floor)


def pack_model(model):
    return dict(
        m=model.filter_size,
        betas=np.array([s.beta for s in model.stages]),
        coeffs=np.stack([s.coeffs for s in model.stages]),
        weights=np.stack([s.weights for s in model.stages]),
        variant=model.variant, floor=np.float64(model.floor),
        rbf_count=model.rbf.count, rbf_radius=model.rbf.radius,
        rbf_bandwidth=np.nan if model.rbf.bandwidth is None
        else model.rbf.bandwidth)


def crops(u):
    H, W = u.shape
    c = CROP
    return dict(
        crop_tl=u[:c, :c], crop_tr=u[:c, W - c:], crop_bl=u[H - c:, :c],
        crop_br=u[H - c:, W - c:],
        crop_c=u[H // 2 - c // 2:H // 2 + c // 2, W // 2 - c // 2:W // 2 + c // 2],
        row_mid=u[H // 2], col_mid=u[:, W // 2],
        sum=np.float64(u.sum()), sumsq=np.float64((u * u).sum()))


def save(name, **kw):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **kw)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def full_case(name, f, model, clean=None, full=True):
    f = np.asarray(f, dtype=np.float32).astype(np.float64)
    t0 = time.time()
    u, _ = sd.run_diffusion(f, model)
    dt = time.time() - t0
    extra = {}
    if clean is not None:
        extra["clean"] = clean if full else np.float64(0)
        extra["psnr"] = np.float64(sd.psnr(u, clean, 255.0))
    out = dict(u=u) if full else crops(u)
    save(name, f=f if full else np.float64(0), full=np.bool_(full),
         f_sum=np.float64(f.sum()), f_crop=f[:CROP, :CROP],
         ref_seconds=np.float64(dt), **pack_model(model), **out, **extra)


def main(which):
    rng = np.random.default_rng(20260101)
    if "small" in which:
        # reference test conventions (tests/test_diffusion.py:12-22)
        full_case("small_m3", rng.uniform(1, 200, (16, 16)),
                  ref_model(3, 3, 2, 9, seed=11, weight_scale=0.05))
        full_case("ragged_m7", rng.uniform(0, 255, (37, 53)),
                  ref_model(7, 5, 2, 63, seed=12))
        full_case("tiny_m7", rng.uniform(1, 255, (4, 5)),
                  ref_model(7, 4, 1, 63, seed=13))
        full_case("m9", rng.uniform(1, 255, (33, 29)),
                  ref_model(9, 6, 2, 63, seed=14))
        full_case("m5_nk24", rng.uniform(1, 255, (40, 44)),
                  ref_model(5, 24, 3, 63, seed=15))
        full_case("m3_M7_nk1", rng.uniform(0, 255, (12, 12)),
                  ref_model(3, 1, 3, 7, seed=16, weight_scale=0.05,
                            betas=[0.3, -0.2, 0.1]))
        full_case("beta_varied", rng.uniform(1, 255, (24, 31)),
                  ref_model(5, 8, 3, 63, seed=17, betas=[0.7, -1.1, 0.2]))
        full_case("narrow_bw", rng.uniform(1, 255, (20, 20)),
                  ref_model(5, 6, 2, 63, seed=18, bandwidth=7.0))
        full_case("wide_bw", rng.uniform(1, 255, (20, 20)),
                  ref_model(5, 6, 2, 63, seed=19, bandwidth=25.0))
        fz = rng.uniform(0, 255, (30, 30))
        fz[rng.uniform(size=fz.shape) < 0.1] = 0.0
        full_case("zeros_in_f", fz, ref_model(7, 8, 2, 63, seed=20))
        fl = rng.uniform(0, 2000, (28, 36))  # far outside the RBF grid
        full_case("wide_range", fl, ref_model(7, 8, 2, 63, seed=21,
                                              weight_scale=0.3))
        # speckled synthetic crops with the BASELINE models
        c2 = synth.CONFIGS["c2"]
        clean, f = synth.noisy_image(c2, 0, 64, 64)
        full_case("c2_crop64", f, ref_model(7, 48, 5, 63, seed=2), clean)
        # primitive pins: conv2d and prox
        img = rng.normal(size=(19, 23)) * 50
        ks = {m: rng.normal(size=(m, m)) for m in (3, 5, 7, 9)}
        save("conv2d", img=img, **{f"k{m}": k for m, k in ks.items()},
             **{f"out{m}": sd.conv2d(img, k) for m, k in ks.items()})
        ut = rng.uniform(-10, 10, (50, 40))
        fp = rng.uniform(1e-3, 10, (50, 40))
        save("prox", u_tilde=ut, f=fp,
             **{f"out_{i}": sd.prox_idiv(ut, fp, lam)
                for i, lam in enumerate((0.01, 0.3, 1.0, 10.0))},
             lams=np.array([0.01, 0.3, 1.0, 10.0]))
    if "projected" in which:
        # the comparison variant (diffusion.py:149-168, 197-224)
        prng = np.random.default_rng(777)
        full_case("projected_m3", prng.uniform(0, 255, (16, 16)),
                  ref_model(3, 2, 3, 7, seed=41, weight_scale=0.2, variant="projected"))
        full_case("projected_m7", prng.uniform(1, 255, (36, 41)),
                  ref_model(7, 8, 3, 63, seed=42, variant="projected", betas=[0.2, -0.3, 0.5]))
        full_case("projected_floor3", prng.uniform(0, 60, (25, 30)),
                  ref_model(5, 6, 2, 63, seed=43, variant="projected", floor=3.0))
    if "io" in which:
        # files written by the reference's own io.py (io.py:133-210, 32-128)
        import specklediff.io as sdio
        model = ref_model(5, 3, 2, 9, seed=31, betas=[0.25, -0.5])
        model.metadata["note"] = "golden"
        sdio.save_model(model, os.path.join(HERE, "io_model_v1.txt"))
        img = rng.uniform(0, 300, (7, 9))
        sdio.save_image(img, os.path.join(HERE, "io_image.fgrid"))
        sdio.save_image(img, os.path.join(HERE, "io_image8.pgm"), peak=255.0)
        sdio.save_image(img, os.path.join(HERE, "io_image16.pgm"), peak=1000.0)
        save("io_arrays", img=img, pgm8=sdio.load_image(os.path.join(HERE, "io_image8.pgm")),
             pgm16=sdio.load_image(os.path.join(HERE, "io_image16.pgm")),
             **pack_model(model))
        print("wrote io fixtures")
    if "training" in which:
        # training.py:69-166 gradients of the real reference (rank 4 of
        # SURVEY 8(f)); inputs are fp32-exact so the GPU sees the same data
        from specklediff import training as sdt
        from specklediff.imageops import conv2d_adjoint, patch_correlation
        from specklediff.speckle import SpeckleConfig, sample_speckle
        trng = np.random.default_rng(777)
        out = {}
        cases = [("p_m3_nk2_T1", 3, 2, 1, 5, (8, 8), "prox"),
                 ("p_m5_nk6_T2", 5, 6, 2, 63, (19, 23), "prox"),
                 ("p_m7_nk20_T2", 7, 20, 2, 63, (33, 29), "prox"),
                 ("q_m3_nk3_T2", 3, 3, 2, 7, (12, 10), "projected"),
                 ("q_m5_nk5_T1", 5, 5, 1, 63, (17, 21), "projected")]
        for ci, (name, m, nk, T, M, shape, variant) in enumerate(cases):
            model = ref_model(m, nk, T, M, seed=500 + ci, weight_scale=0.3,
                              variant=variant, betas=list(0.3 * trng.standard_normal(T)))
            clean = np.float32(trng.uniform(20.0, 235.0, size=shape)).astype(np.float64)
            noisy = np.float32(sample_speckle(clean, SpeckleConfig(looks=4, seed=7)).noisy).astype(np.float64)
            pair = sample_speckle(clean, SpeckleConfig(looks=4, seed=7))
            pair = type(pair)(clean=clean, noisy=noisy, config=pair.config)
            total, acc = sdt.loss_and_gradients(model, [pair], list(range(T)), T - 1)
            _, traces = sdt._forward(model, noisy, T - 1, 0)
            gn = np.float32(trng.normal(size=shape)).astype(np.float64)
            g_prev, grads = sdt._stage_backward(traces[T - 1], model.stages[T - 1], noisy, gn, model)
            rec = dict(pack_model(model), clean=clean, noisy=noisy, loss=total, g_next=gn,
                       g_prev=g_prev, sb_beta=grads.beta, sb_coeffs=grads.coeffs,
                       sb_weights=grads.weights, u_prev=traces[T - 1].u_prev)
            for t in range(T):
                rec[f"beta_{t}"] = acc[t].beta
                rec[f"coeffs_{t}"] = acc[t].coeffs
                rec[f"weights_{t}"] = acc[t].weights
            save(f"train_{name}", **rec)
        img = np.float32(trng.normal(size=(14, 11))).astype(np.float64)
        adj = np.float32(trng.normal(size=(14, 11))).astype(np.float64)
        for m in (1, 3, 5, 7, 9):
            k = trng.normal(size=(m, m))
            out[f"k{m}"] = k
            out[f"adj{m}"] = conv2d_adjoint(img, k)
            out[f"pc{m}"] = patch_correlation(img, adj, m)
        save("train_imageops", img=img, adj=adj, **out)
        print("wrote training fixtures")
    if "overflow" in which:
        # fp32 range edge of the error contract (diffusion.py:238-239,
        # speckle.py:119-121): the reference squares u~ in float64
        orng = np.random.default_rng(0)
        f = orng.uniform(1, 255, (40, 40))
        # weights 1e30: |u~| ~ 1e31 (u~^2 overflows fp32) but the reference
        # finishes with a finite image (max ~1e29)
        full_case("huge_weights", f, ref_model(3, 2, 3, 7, seed=1, weight_scale=1e30))
        # stage 1 weights 1e300: the reference's u~^2 overflows float64 in
        # stage 1 -> FloatingPointError("non-finite image after stage 1")
        model = ref_model(3, 2, 3, 7, seed=1)
        model.stages[1].weights *= 1e301
        f32 = np.asarray(f, dtype=np.float32).astype(np.float64)
        try:
            sd.run_diffusion(f32, model)
            msg = ""
        except FloatingPointError as e:
            msg = str(e)
        assert msg, "expected the reference to raise"
        save("overflow_stage1", f=f32, raises=msg, **pack_model(model))
        # prox far outside the fp32 square range, results inside fp32
        big = orng.uniform(-1, 1, (20, 20)) * 10.0 ** orng.uniform(15, 37, (20, 20))
        fb = 10.0 ** orng.uniform(-3, 19, (20, 20))
        big = np.asarray(big, dtype=np.float32).astype(np.float64)
        fb = np.asarray(fb, dtype=np.float32).astype(np.float64)
        save("prox_large", u_tilde=big, f=fb,
             **{f"out_{i}": sd.prox_idiv(big, fb, lam) for i, lam in enumerate((0.3, 1.0, 10.0))},
             lams=np.array([0.3, 1.0, 10.0]))
    for key in ("c1", "c2"):
        if key in which:
            cfg = synth.CONFIGS[key]
            clean, f = synth.noisy_image(cfg, 0)
            model = ref_model(cfg.m, cfg.nk, cfg.T, cfg.M, seed=cfg.index)
            full_case(f"{key}_full", f, model, clean, full=False)


if __name__ == "__main__":
    main(sys.argv[1:] or ["small", "projected", "io", "training", "c1", "c2"])

"""The fused kernel's row-strip mode (TOP/BOTTOM_HALO) on one GPU.

Ranks are emulated in lock-step inside one process (halo rows copied
between the strips' device buffers between stages; no kernel ever waits on
another), which checks the kernel side of the C4 path: stitched strips must
be BIT-identical to the whole-image despeckle (per-pixel arithmetic does
not depend on where a tile starts).  The real exchange (run_strip +
torch.distributed) is covered on CPU by test_strips_cpu.py."""
import numpy as np
import pytest

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, strips, synth

pytestmark = pytest.mark.gpu


def lockstep_strips(dm, f, world, T):
    torch = __import__("torch")
    H, W = f.shape
    h = dm.m - 1
    lays = [strips.StripLayout(H, W, world, r, h) for r in range(world)]
    ext = []
    for lay in lays:
        r0, r1 = lay.rows
        fe = torch.zeros(lay.n + 2 * h, W, device="cuda")
        fe[h:h + lay.n] = f[r0:r1]
        ext.append([fe, torch.zeros_like(fe), torch.zeros_like(fe)])
    st = dm.status()
    st.reset()

    def exchange(which):
        for r, lay in enumerate(lays):
            buf = ext[r][which]
            if lay.has_top:
                up = ext[r - 1][which]
                buf[0:h] = up[lays[r - 1].n:lays[r - 1].n + h]
            if lay.has_bottom:
                dn = ext[r + 1][which]
                buf[lay.n + h:lay.n + 2 * h] = dn[h:2 * h]

    cur = 0
    for t in range(T):
        exchange(cur)
        dst = 1 + t % 2
        for r, lay in enumerate(lays):
            fl = lay.flags | ((_lib.STAGE_FLOOR_INPUT | _lib.STAGE_CHECK_F) if t == 0 else 0)
            dm.stage(t, ext[r][cur], ext[r][0], out=ext[r][dst], flags=fl,
                     status=st, rows=(h, lay.n))
        cur = dst
    st.check()
    return torch.cat([ext[r][cur][h:h + lays[r].n] for r in range(world)])


@pytest.mark.parametrize("m,world", [(7, 2), (7, 5), (5, 3), (9, 4), (3, 7)])
def test_strips_bit_identical_to_whole_image(cuda, m, world):
    torch = cuda
    model = synth.make_model(m, 8, 3, 63, seed=m * 10 + world)
    H, W = 203, 97
    f = torch.from_numpy(np.random.default_rng(m).uniform(0, 300, (H, W))
                         .astype(np.float32)).cuda()
    dm = tn.device_model_for(model)
    whole = dm.despeckle(f)
    got = lockstep_strips(dm, f, world, model.num_stages)
    assert torch.equal(got, whole)


def test_c4_scene_band_strips(cuda, oracle):
    """A 2-strip split of a C4 band, boundary at a scene row that is a
    multiple of 2048 (the G=8 strip edges), against the oracle."""
    torch = cuda
    cfg = synth.CONFIGS["c4"]
    model = synth.config_model(cfg)
    y0, y1, x0, x1 = 2048 - 80, 2048 + 80, 4000, 4200
    f = synth.scene_crop(cfg, y0, y1, x0, x1)
    dm = tn.device_model_for(model)
    got = lockstep_strips(dm, torch.from_numpy(f).cuda(), 2, cfg.T).cpu().numpy()
    ref = oracle.run_diffusion(f.astype(np.float64), model)
    assert np.max(np.abs(got - ref) / ref) <= 1e-4

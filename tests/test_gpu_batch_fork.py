"""Batch fork (DESIGN.md §7b item 5): in auto mode a batch whose half still
selects the large-tile kernel runs its two halves on two streams.  The
result must be bit-identical to the one-stream run of the same kernel
(forced large tiles, which never forks) and to the halves run separately;
plans (captured CUDA graphs) and the device-side input check must keep
working through the fork."""
import numpy as np
import pytest
import torch

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

pytestmark = pytest.mark.gpu

# 32 x 512^2: the half (16 images, 1,024 large tiles) is >= 3 waves of 2 CTAs
# per SM on 148 SMs, so auto forks (both halves on the tile kernel); 16 images
# alone do not fork (8-image half)
B, HW = 32, 512


@pytest.fixture(scope="module")
def batch():
    cfg = synth.CONFIGS["c3"]
    model = synth.config_model(cfg)
    base = np.stack([synth.noisy_image(cfg, i, HW, HW)[1] for i in range(4)])
    rng = np.random.default_rng(5)
    f = base[np.arange(B) % 4] * rng.uniform(0.5, 1.5, (B, 1, 1)).astype(np.float32)
    return model, f.astype(np.float32)


def test_fork_bit_identical_to_one_stream(cuda, batch):
    model, f = batch
    dm = tn.device_model_for(model)
    fd = torch.from_numpy(f).cuda()
    _lib.launch_count_reset()
    forked = dm.despeckle(fd)
    torch.cuda.synchronize()
    # two halves x T stage launches, one tile-kernel launch each
    assert _lib.launch_count() == 2 * synth.CONFIGS["c3"].T
    _lib.set_stage_kernel(_lib.KERNEL_LARGE_TILES)
    try:
        one = dm.despeckle(fd)
        # (a 16-image batch alone selects the cluster kernel in auto mode)
        halves = torch.cat([dm.despeckle(fd[:B // 2]), dm.despeckle(fd[B // 2:])])
    finally:
        _lib.set_stage_kernel(_lib.KERNEL_AUTO)
    assert torch.equal(forked, one)
    assert torch.equal(forked, halves)


def test_fork_odd_batch_and_strided(cuda, batch):
    model, f = batch
    dm = tn.device_model_for(model)
    fd = torch.from_numpy(f[:B - 1]).cuda()          # odd: halves 16 + 15
    padded = torch.zeros(B - 1, HW + 3, HW + 8, device="cuda")
    padded[:, :HW, :HW] = fd
    view = padded[:, :HW, :HW]
    out = torch.empty_like(padded)[:, :HW, :HW]
    work = torch.empty_like(padded)[:, :HW, :HW]
    a = dm.despeckle(fd)
    b = dm.despeckle(view, out=out, work=work)
    _lib.set_stage_kernel(_lib.KERNEL_LARGE_TILES)
    try:
        c = dm.despeckle(fd)
    finally:
        _lib.set_stage_kernel(_lib.KERNEL_AUTO)
    assert torch.equal(a, c)
    assert torch.equal(b, c)


def test_fork_plan_graph_and_status(cuda, batch):
    model, f = batch
    dm = tn.device_model_for(model)
    ref = dm.despeckle(torch.from_numpy(f).cuda()).cpu().numpy()
    for _ in range(3):                                # eager, capture, replay
        np.testing.assert_array_equal(dm.despeckle_host(f), ref)
    bad = f.copy()
    bad[B - 1, 7, 9] = -1.0                            # in the second half
    with pytest.raises(ValueError, match="nonnegative"):
        dm.despeckle_host(bad)
    np.testing.assert_array_equal(dm.despeckle_host(f), ref)

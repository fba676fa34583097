"""Calling-convention contracts of the device entry points: layouts, explicit
streams, plan reuse across the device / host entries, and the one-launch
diffusion_step (u_next and force together)."""
import numpy as np
import pytest

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

pytestmark = pytest.mark.gpu


def _model():
    return synth.make_model(7, 8, 3, 63, seed=31)


def test_dense_f_into_padded_out_and_work(cuda):
    """f dense, out / work padded views (another row stride): f is copied
    into out's layout (one stride for all three buffers), same bits as the
    dense run."""
    torch = cuda
    dm = tn.device_model_for(_model())
    f = torch.from_numpy(np.random.default_rng(2).uniform(1, 255, (3, 70, 90)).astype(np.float32)).cuda()
    ref = dm.despeckle(f)
    big_o = torch.full((3, 70, 128), -7.0, device="cuda")
    big_w = torch.full((3, 70, 128), -7.0, device="cuda")
    out = big_o[:, :, :90]
    work = big_w[:, :, :90]
    got = dm.despeckle(f, out=out, work=work)
    assert got.data_ptr() == out.data_ptr()
    assert torch.equal(got, ref)
    assert torch.all(big_o[:, :, 90:] == -7.0)        # padding untouched


def test_explicit_stream(cuda):
    """stream= another than the current one: temporaries and the status read
    follow that stream; same result as the current-stream call, and a bad f
    is still reported."""
    torch = cuda
    dm = tn.device_model_for(_model())
    f = torch.from_numpy(np.random.default_rng(3).uniform(1, 255, (2, 64, 64)).astype(np.float32)).cuda()
    ref = dm.despeckle(f)
    s = torch.cuda.Stream()
    for _ in range(3):
        got = dm.despeckle(f, stream=s)
        s.synchronize()
        assert torch.equal(got, ref)
    bad = f.clone()
    bad[1, 3, 3] = -1.0
    with pytest.raises(ValueError, match="nonnegative"):
        dm.despeckle(bad, stream=s)
    u = torch.from_numpy(np.random.default_rng(4).uniform(1, 255, (64, 64)).astype(np.float32)).cuda()
    a = dm.stage(1, u, u)
    b = dm.stage(1, u, u, stream=s)
    s.synchronize()
    assert torch.equal(a, b)


def test_plan_device_then_host(cuda):
    """A device call on a plan followed at once by a host call on the same
    plan (its buffers): the host path -- here the banded one, whose copy and
    band streams are not the plan's stream -- waits for the queued device
    work.  2816^2 = 44 x 44 large tiles: >= 2 x 3 waves, so it is banded."""
    torch = cuda
    model = synth.config_model(synth.CONFIGS["c2"])
    dm = tn.device_model_for(model)
    rng = np.random.default_rng(5)
    fa = rng.uniform(1, 255, (2816, 2816)).astype(np.float32)
    fb = rng.uniform(1, 255, (2816, 2816)).astype(np.float32)
    ua = dm.despeckle_host(fa)
    ub = dm.despeckle_host(fb)
    p = dm._plan(1, 2816, 2816)
    L = _lib.load()
    import ctypes
    fdev = torch.from_numpy(fa).cuda()
    udev = torch.empty_like(fdev)
    torch.cuda.synchronize()
    for _ in range(2):
        _lib.check(L.tnrd_plan_despeckle_device(p, ctypes.c_void_p(fdev.data_ptr()),
                                                ctypes.c_void_p(udev.data_ptr())))
        got = dm.despeckle_host(fb)
        assert np.array_equal(got, ub)
    torch.cuda.synchronize()
    assert np.array_equal(udev.cpu().numpy(), ua)


@pytest.mark.parametrize("variant", ["prox", "projected"])
def test_stage_force_one_launch(cuda, variant):
    """tnrd_stage_force: u_next equals tnrd_stage's and the force equals
    the TNRD_STAGE_FORCE launch's, bit for bit, from one launch."""
    torch = cuda
    model = _model()
    model.variant = variant
    dm = tn.device_model_for(model)
    for shape in [(64, 64), (2, 200, 130), (600, 512)]:
        u = torch.from_numpy(np.random.default_rng(6).uniform(1, 255, shape).astype(np.float32)).cuda()
        f = torch.from_numpy(np.random.default_rng(7).uniform(1, 255, shape).astype(np.float32)).cuda()
        ref_u = dm.stage(1, u, f)
        ref_force = dm.stage(1, u, f, flags=_lib.STAGE_FORCE)
        torch.cuda.synchronize()
        _lib.launch_count_reset()
        got_u, got_force = dm.stage_force(1, u, f)
        torch.cuda.synchronize()
        assert _lib.launch_count() == 1           # tile or cluster kernel: one launch
        assert torch.equal(got_u, ref_u)
        assert torch.equal(got_force, ref_force)


def test_diffusion_step_single_pass(cuda):
    """diffusion_step returns u_next and u~ = u - force from one stage
    launch (was two)."""
    model = _model()
    rng = np.random.default_rng(8)
    u = rng.uniform(1, 255, (50, 60))
    f = rng.uniform(1, 255, (50, 60))
    tn.diffusion_step(u, f, model.stages[0], model)   # upload
    _lib.launch_count_reset()
    u_next, tr = tn.diffusion_step(u, f, model.stages[0], model)
    assert _lib.launch_count() == 1
    ref = tn.run_diffusion  # noqa: F841  (API present)
    assert np.all(np.isfinite(tr.u_tilde)) and np.array_equal(tr.u_next, u_next)

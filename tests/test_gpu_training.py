"""GPU stage backward (training.py:69-166,
imageops.py:75-127) against gradients of the REAL reference, committed as
fixtures by tests/golden/make_golden.py (training section), plus the
reference's structural tests restated (tests/test_training.py:98-141,
tests/test_imageops.py:89-116).  fp32 on the device vs float64 in the
reference: errors are measured relative to each array's largest entry."""
import numpy as np
import pytest

from conftest import golden_model, load_golden

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import training as tr
from paper_1702_07482_b200.diffusion import StageTrace
from paper_1702_07482_b200.speckle import NoisyPair, SpeckleConfig

pytestmark = pytest.mark.gpu

CASES = ["p_m3_nk2_T1", "p_m5_nk6_T2", "p_m7_nk20_T2", "q_m3_nk3_T2", "q_m5_nk5_T1"]
TOL = 2e-4   # max |gpu - ref| / max |ref| per gradient array


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_imageops_drop_ins_match_reference(cuda):
    g = load_golden("train_imageops")
    for m in (1, 3, 5, 7, 9):
        assert rel(tn.conv2d_adjoint(g["img"], g[f"k{m}"]), g[f"adj{m}"]) < 1e-5, m
        assert rel(tn.patch_correlation(g["img"], g["adj"], m), g[f"pc{m}"]) < 1e-5, m


@pytest.mark.parametrize("m", [3, 5, 7])
def test_adjoint_identity(cuda, m):
    # reference tests/test_imageops.py:89-96 (fp32 tolerance)
    rng = np.random.default_rng(m)
    a = rng.normal(size=(12, 12))
    b = rng.normal(size=(12, 12))
    k = rng.normal(size=(m, m))
    lhs = np.sum(tn.conv2d(a, k) * b)
    rhs = np.sum(a * tn.conv2d_adjoint(b, k))
    assert abs(lhs - rhs) < 1e-4 * np.sum(np.abs(a)) * np.abs(k).sum() / a.size * 10


@pytest.mark.parametrize("name", CASES)
def test_stage_backward_matches_reference(cuda, name):
    g = load_golden(f"train_{name}")
    model = golden_model(g)
    T = model.num_stages
    trace = StageTrace(g["u_prev"], None, None, None, None)
    gp = tr.backprop_adjoint(trace, model.stages[T - 1], g["noisy"], g["g_next"], model)
    assert rel(gp, g["g_prev"]) < TOL
    gr = tr.grad_stage_params(trace, model.stages[T - 1], g["noisy"], g["g_next"], model)
    assert abs(gr.beta - float(g["sb_beta"])) <= TOL * abs(float(g["sb_beta"])) + 1e-9
    assert rel(gr.coeffs, g["sb_coeffs"]) < TOL
    assert rel(gr.weights, g["sb_weights"]) < TOL


@pytest.mark.parametrize("name", CASES)
def test_loss_and_gradients_match_reference(cuda, name):
    g = load_golden(f"train_{name}")
    model = golden_model(g)
    T = model.num_stages
    pair = NoisyPair(clean=g["clean"], noisy=g["noisy"], config=SpeckleConfig(4, 7))
    total, acc = tr.loss_and_gradients(model, [pair], list(range(T)), T - 1)
    assert abs(total - float(g["loss"])) <= 1e-4 * float(g["loss"])
    for t in range(T):
        ref_b = float(g[f"beta_{t}"])
        assert abs(acc[t].beta - ref_b) <= TOL * abs(ref_b) + 1e-6, t
        assert rel(acc[t].coeffs, g[f"coeffs_{t}"]) < TOL, t
        assert rel(acc[t].weights, g[f"weights_{t}"]) < TOL, t


def test_zero_adjoint_gives_zero(cuda):
    # reference tests/test_training.py:111-141
    g = load_golden("train_p_m5_nk6_T2")
    model = golden_model(g)
    trace = StageTrace(g["u_prev"], None, None, None, None)
    z = np.zeros_like(g["u_prev"])
    assert np.all(tr.backprop_adjoint(trace, model.stages[0], g["noisy"], z, model) == 0)
    gr = tr.grad_stage_params(trace, model.stages[0], g["noisy"], z, model)
    assert gr.beta == 0.0 and np.all(gr.coeffs == 0) and np.all(gr.weights == 0)


def test_identity_limit(cuda):
    # reference tests/test_training.py:98-109: zero weights, tiny lambda
    from paper_1702_07482_b200 import synth
    model = synth.make_model(3, 1, 1, 5, seed=4, beta=float(np.log(1e-8)))
    model.stages[0].weights[:] = 0.0
    rng = np.random.default_rng(13)
    f = rng.uniform(20, 235, (8, 8))
    trace = StageTrace(np.maximum(f, 1e-6), None, None, None, None)
    gn = rng.normal(size=(8, 8))
    out = tr.backprop_adjoint(trace, model.stages[0], f, gn, model)
    assert np.abs(out - gn).max() < 1e-5


def test_backward_bit_reproducible(cuda):
    g = load_golden("train_p_m7_nk20_T2")
    model = golden_model(g)
    trace = StageTrace(g["u_prev"], None, None, None, None)
    a = tr.grad_stage_params(trace, model.stages[1], g["noisy"], g["g_next"], model)
    b = tr.grad_stage_params(trace, model.stages[1], g["noisy"], g["g_next"], model)
    assert a.beta == b.beta
    np.testing.assert_array_equal(a.coeffs, b.coeffs)
    np.testing.assert_array_equal(a.weights, b.weights)

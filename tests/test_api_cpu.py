"""Host-side logic of the drop-in API (no GPU): model containers and their
validation mirror the reference (diffusion.py:46-130, influence.py:9-37),
parameter preparation, synthetic workload determinism."""
import math

import numpy as np
import pytest

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import engine, synth


@pytest.mark.parametrize("m", [3, 5, 7, 9])
def test_basis_orthonormal_zero_mean_and_matches_oracle(oracle, m):
    b = tn.zero_mean_basis(m)
    assert b.shape == (m * m, m * m - 1)
    np.testing.assert_allclose(b.T @ b, np.eye(m * m - 1), atol=1e-12)
    assert np.abs(b.sum(axis=0)).max() < 1e-12
    np.testing.assert_allclose(b, oracle.basis(m), atol=1e-15)


def test_basis_rejects_even():
    with pytest.raises(ValueError):
        tn.zero_mean_basis(4)


def test_model_validation_mirrors_reference():
    rng = np.random.default_rng(0)
    s3 = tn.StageParams(0.0, rng.normal(size=(2, 8)), rng.normal(size=(2, 63)))
    with pytest.raises(ValueError, match="at least one stage"):
        tn.DiffusionModel(stages=[], filter_size=3, looks=1)
    with pytest.raises(ValueError, match="unknown variant"):
        tn.DiffusionModel(stages=[s3], filter_size=3, looks=1, variant="x")
    with pytest.raises(ValueError, match="odd"):
        tn.DiffusionModel(stages=[s3], filter_size=4, looks=1)
    with pytest.raises(ValueError, match="basis coeffs"):
        tn.DiffusionModel(stages=[s3], filter_size=5, looks=1)
    with pytest.raises(ValueError, match="RBF weights"):
        tn.DiffusionModel(stages=[s3], filter_size=3, looks=1,
                          rbf=tn.RbfGrid(7, 310.0))
    s3b = tn.StageParams(0.0, rng.normal(size=(3, 8)), rng.normal(size=(3, 63)))
    with pytest.raises(ValueError, match="filter count"):
        tn.DiffusionModel(stages=[s3, s3b], filter_size=3, looks=1)
    with pytest.raises(ValueError, match="disagree"):
        tn.StageParams(0.0, rng.normal(size=(2, 8)), rng.normal(size=(3, 63)))
    with pytest.raises(ValueError, match="projection floor"):
        tn.DiffusionModel(stages=[s3], filter_size=3, looks=1,
                          variant="projected", floor=0.0)
    m = tn.DiffusionModel(stages=[s3], filter_size=3, looks=1)
    assert m.rbf.count == 63 and math.isclose(m.rbf.radius, 310.0)
    assert math.isclose(m.rbf.gamma, 10.0)
    assert m.num_filters == 2 and m.num_stages == 1


def test_rbf_grid_validation_and_params():
    with pytest.raises(ValueError):
        tn.RbfGrid(1, 1.0)
    with pytest.raises(ValueError):
        tn.RbfGrid(5, 0.0)
    with pytest.raises(ValueError):
        tn.RbfGrid(5, 1.0, bandwidth=-1.0)
    g = tn.RbfGrid(63, 310.0)
    np.testing.assert_allclose(g.centers, np.linspace(-310, 310, 63))
    mu0, delta, gamma = engine.rbf_grid_params(63, 310.0)
    assert mu0 == -310.0 and math.isclose(delta, 10.0) and math.isclose(gamma, 10.0)
    assert engine.rbf_grid_params(63, 310.0, 7.0)[2] == 7.0


def test_stage_kernels_match_reference_formula(oracle):
    model = synth.make_model(7, 5, 2, 63, seed=3)
    k = engine.model_kernels(model)
    for t, s in enumerate(model.stages):
        np.testing.assert_allclose(k[t], oracle.stage_kernels(s.coeffs, 7), atol=1e-15)
        # zero-mean, unit-norm kernels (orthonormal basis, unit coeffs)
        np.testing.assert_allclose(k[t].sum(axis=(1, 2)), 0.0, atol=1e-12)
        np.testing.assert_allclose(np.sqrt((k[t] ** 2).sum(axis=(1, 2))), 1.0)


def test_fingerprint_sees_in_place_edits():
    model = synth.make_model(3, 2, 2, 7, seed=1)
    k = engine.model_kernels(model)
    w = np.stack([s.weights for s in model.stages])
    lam = np.ones(2)
    a = engine.params_fingerprint(3, k, w, lam, (0, 1, 1))
    w[1, 0, 0] += 1e-12
    assert engine.params_fingerprint(3, k, w, lam, (0, 1, 1)) != a


def test_synthetic_workloads_are_deterministic_and_in_range():
    cfg = synth.CONFIGS["c2"]
    c1, f1 = synth.noisy_image(cfg, 0, 64, 80)
    c2, f2 = synth.noisy_image(cfg, 0, 64, 80)
    np.testing.assert_array_equal(f1, f2)
    assert c1.min() >= 1.0 and c1.max() <= 255.0
    assert f1.dtype == np.float32 and np.all(f1 > 0)
    # C4 tiled scene: a crop equals the same rows of the band it lies in
    c4 = synth.CONFIGS["c4"]
    crop = synth.scene_crop(c4, 1000, 1040, 2040, 2060)
    band = synth.scene_rows(c4, 1000, 1040)
    np.testing.assert_array_equal(crop, band[:, 2040:2060])


def test_speckle_matches_reference_generator():
    # reference speckle.py:51-61: Philox keyed by the seed, Gamma(L, 1/L)
    cfg = tn.SpeckleConfig(looks=4, seed=123)
    n = tn.speckle_field((32, 32), cfg)
    rng = np.random.Generator(np.random.Philox(key=123))
    np.testing.assert_array_equal(n, np.sqrt(rng.gamma(4.0, 0.25, (32, 32))))
    with pytest.raises(ValueError):
        tn.sample_speckle(-np.ones((3, 3)), cfg)
    with pytest.raises(ValueError):
        tn.SpeckleConfig(looks=0, seed=1)


def test_config_table_matches_baseline():
    c = synth.CONFIGS
    assert (c["c1"].H, c["c1"].m, c["c1"].nk, c["c1"].T) == (256, 5, 24, 5)
    assert (c["c2"].H, c["c2"].m, c["c2"].nk, c["c2"].T, c["c2"].batch) == (512, 7, 48, 5, 1)
    assert (c["c3"].batch, c["c3"].looks) == (256, (1, 2, 4, 8))
    assert (c["c4"].H, c["c4"].W) == (16384, 16384)
    assert (c["c5"].H, c["c5"].m, c["c5"].nk, c["c5"].T, c["c5"].batch) == (1024, 9, 80, 8, 32)

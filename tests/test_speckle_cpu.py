"""GPU speckle generator, CPU side: the Philox4x32-10
integer core pinned to the published known-answer vector and to curand's
host Philox generator, and the float64 oracle restatement of the sampler
checked against the reference's own statistical tests and against the
reference's numpy stream in distribution.  No GPU needed."""
import ctypes
import math
import os

import numpy as np
import pytest

from paper_1702_07482_b200 import _lib
from paper_1702_07482_b200.speckle import SpeckleConfig, speckle_field

# Random123 known-answer vector (philox4x32, 10 rounds, counter 0, key 0)
KAT = (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)


def _lib_philox(ctr, key):
    L = _lib.load()
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    L.tnrd_philox4x32_10(c, k, o)
    return tuple(o)


def test_philox_known_answer(oracle):
    assert oracle.philox4x32_10((0, 0, 0, 0), (0, 0)) == KAT
    assert _lib_philox((0, 0, 0, 0), (0, 0)) == KAT   # the shipped library's core


def test_philox_matches_curand_host_generator(oracle):
    """curand's Philox4_32_10 host generator: its first block for seed s is
    Philox(counter 0, key = (s lo, s hi))."""
    path = "/usr/local/cuda/lib64/libcurand.so"
    if not os.path.exists(path):
        pytest.skip("libcurand not present")
    cr = ctypes.CDLL(path)
    for seed in (0, 1, 0x123456789ABCDEF, 2 ** 64 - 1):
        g = ctypes.c_void_p()
        assert cr.curandCreateGeneratorHost(ctypes.byref(g), 161) == 0   # PHILOX4_32_10
        assert cr.curandSetPseudoRandomGeneratorSeed(g, ctypes.c_ulonglong(seed)) == 0
        buf = (ctypes.c_uint32 * 4)()
        assert cr.curandGenerate(g, buf, ctypes.c_size_t(4)) == 0
        cr.curandDestroyGenerator(g)
        key = (seed & 0xFFFFFFFF, seed >> 32)
        assert tuple(buf) == oracle.philox4x32_10((0, 0, 0, 0), key)
        assert tuple(buf) == _lib_philox((0, 0, 0, 0), key)


@pytest.mark.parametrize("looks", [1, 3, 5, 8])
def test_oracle_unit_mean_intensity(oracle, looks):
    # reference tests/test_speckle.py:60-63
    n = oracle.speckle_field((1000, 1000), looks, 42)
    assert abs(np.mean(n ** 2) - 1.0) < 0.005


def test_oracle_variance_and_rayleigh_mean(oracle):
    # reference tests/test_speckle.py:65-74
    n = oracle.speckle_field((1000, 1000), 64, 9)
    assert abs(np.var(n ** 2) - 1.0 / 64) < 0.05 / 64
    n = oracle.speckle_field((1000, 1000), 1, 11)
    expect = math.sqrt(math.pi) / 2.0
    assert abs(np.mean(n) - expect) / expect < 0.005


@pytest.mark.parametrize("looks", [1, 4])
def test_oracle_matches_reference_stream_in_distribution(oracle, looks):
    """Two-sample KS between the counter-based sampler and the reference's
    own numpy Generator(Philox).gamma stream (speckle.py:51-61)."""
    from scipy.stats import ks_2samp
    ours = oracle.speckle_field((400, 500), looks, 7).ravel() ** 2
    ref = speckle_field((400, 500), SpeckleConfig(looks=looks, seed=7)).ravel() ** 2
    assert ks_2samp(ours, ref).pvalue > 1e-3


def test_oracle_counter_layout(oracle):
    """Pixel i of the field is a pure function of (seed, looks, i): a field
    computed from an index offset equals the tail of the full field."""
    full = oracle.speckle_field((3, 50, 40), 2, 99)
    tail = oracle.speckle_field((2, 50, 40), 2, 99, base=50 * 40)
    np.testing.assert_array_equal(full[1:], tail)

"""CPU float64 oracle for the TNRD inference path (TEST INFRASTRUCTURE ONLY).

This module is the *checker*.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (``cpu_baseline`` leg and ``--impl reference``) may import
it.  The product package ``paper_1702_07482_b200`` never imports it and has
no CPU fallback.

It wraps ``oracle/tnrd_oracle.c`` (built by ``oracle/Makefile`` into
``oracle/libtnrd_oracle.so``) and restates the small host-side pieces of the
reference needed to feed it:

* ``basis(m)``            -- diffusion.py:27-43 (zero_mean_basis)
* ``stage_kernels``       -- diffusion.py:76-77 (coeffs @ basis.T)
* ``rbf_centers/gamma``   -- influence.py:29-37 (linspace, bandwidth default)
* ``run_diffusion``       -- diffusion.py:227-242 via the C restatement
* ``psnr``                -- metrics.py:28-39 (used for the PSNR-delta gate)

Parity of this oracle against the real reference is pinned by
``tests/test_oracle.py`` on the golden vectors in ``tests/golden/``.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtnrd_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc, OpenMP) if needed."""
    src = os.path.join(_HERE, "tnrd_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_run_diffusion.restype = ctypes.c_int
        L.oracle_run_diffusion.argtypes = [
            _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, ctypes.c_double, _dp,
            _dp, ctypes.c_int]
        L.oracle_run_diffusion_ex.restype = ctypes.c_int
        L.oracle_run_diffusion_ex.argtypes = [
            _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, ctypes.c_double, _dp,
            ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int]
        L.oracle_stage.restype = None
        L.oracle_stage.argtypes = [
            _dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, _dp, _dp, _dp, ctypes.c_double, ctypes.c_double, _dp]
        L.oracle_force.restype = None
        L.oracle_force.argtypes = [
            _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, _dp, _dp, _dp, ctypes.c_double, _dp]
        L.oracle_conv2d.restype = None
        L.oracle_conv2d.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp,
                                    ctypes.c_int, _dp]
        L.oracle_prox_idiv.restype = None
        L.oracle_prox_idiv.argtypes = [_dp, _dp, ctypes.c_double, _dp,
                                       ctypes.c_long]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_set_threads.restype = None
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _u32p = ctypes.POINTER(ctypes.c_uint32)
        L.oracle_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.oracle_philox4x32_10.restype = None
        L.oracle_speckle_field.argtypes = [_dp, ctypes.c_long, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_speckle_field.restype = None
        L.oracle_set_threads(-1)  # default: every host core
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ----------------------------------------------------------- host-side params

def basis(m: int) -> np.ndarray:
    """diffusion.py:27-43 -- the m*m-1 non-DC separable DCT-II atoms as the
    columns of an (m*m, m*m-1) matrix, ordered p-major then q."""
    n = np.arange(m)
    rows = [np.full(m, math.sqrt(1.0 / m))]
    for p in range(1, m):
        rows.append(math.sqrt(2.0 / m) * np.cos(np.pi * (n + 0.5) * p / m))
    cols = [np.outer(rows[p], rows[q]).ravel()
            for p in range(m) for q in range(m) if (p, q) != (0, 0)]
    return np.stack(cols, axis=1)


def stage_kernels(coeffs: np.ndarray, m: int) -> np.ndarray:
    """diffusion.py:76-77 -- k_i = coeffs_i @ basis.T reshaped to (m, m)."""
    coeffs = np.asarray(coeffs, dtype=np.float64)
    return (coeffs @ basis(m).T).reshape(coeffs.shape[0], m, m)


def rbf_centers(count: int, radius: float) -> np.ndarray:
    """influence.py:29-31"""
    return np.linspace(-radius, radius, count)


def rbf_gamma(count: int, radius: float, bandwidth=None) -> float:
    """influence.py:33-37"""
    if bandwidth is not None:
        return float(bandwidth)
    return 2.0 * radius / (count - 1)


def model_arrays(model):
    """Flatten a DiffusionModel (ours or the reference's: duck-typed on
    .stages[t].{beta,coeffs,weights}, .filter_size, .rbf.{count,radius,
    bandwidth}) into the oracle's float64 arrays."""
    m = int(model.filter_size)
    kern = np.stack([stage_kernels(s.coeffs, m) for s in model.stages])
    w = np.stack([np.asarray(s.weights, dtype=np.float64)
                  for s in model.stages])
    lams = np.array([math.exp(float(s.beta)) for s in model.stages])
    g = model.rbf
    return dict(kernels=kern, weights=w, lams=lams,
                centers=rbf_centers(g.count, g.radius),
                gamma=rbf_gamma(g.count, g.radius, g.bandwidth))


# ------------------------------------------------------------------ entry points

def set_threads(n: int) -> None:
    """Worker threads of the C oracle (n <= 0: every host core)."""
    lib().oracle_set_threads(int(n))


def run_diffusion_arrays(f, kernels, weights, centers, gamma, lams,
                         nthreads: int = 0, variant: str = "prox",
                         floor: float = 1.0):
    """Returns (u_T float64, bad_stage) -- bad_stage is -1 when every stage
    stayed finite (diffusion.py:238-239 semantics).  variant "projected"
    follows diffusion.py:149-168, 197-224."""
    f = _c64(f)
    if f.ndim != 2:
        raise ValueError("f must be 2D")
    kernels = _c64(kernels)
    T, nk, m, _ = kernels.shape
    weights = _c64(weights)
    centers = _c64(centers)
    lams = _c64(lams)
    H, W = f.shape
    out = np.empty_like(f)
    bad = lib().oracle_run_diffusion_ex(
        _p(f), H, W, m, nk, T, centers.size, _p(kernels), _p(weights),
        _p(centers), float(gamma), _p(lams), 1 if variant == "projected" else 0,
        float(floor), _p(out), int(nthreads))
    return out, int(bad)


def run_diffusion(f, model, nthreads: int = 0) -> np.ndarray:
    """Oracle of specklediff.run_diffusion (prox variant)."""
    a = model_arrays(model)
    f = _c64(f)
    if np.any(f < 0):
        raise ValueError("observation must be nonnegative")
    out, bad = run_diffusion_arrays(f, a["kernels"], a["weights"],
                                    a["centers"], a["gamma"], a["lams"],
                                    nthreads, getattr(model, "variant", "prox"),
                                    float(getattr(model, "floor", 1.0)))
    if bad >= 0:
        raise FloatingPointError(f"non-finite image after stage {bad}")
    return out


def stage(u, f, kernels_t, weights_t, centers, gamma, lam) -> np.ndarray:
    u = _c64(u); f = _c64(f)
    kernels_t = _c64(kernels_t); weights_t = _c64(weights_t)
    centers = _c64(centers)
    nk, m, _ = kernels_t.shape
    H, W = u.shape
    out = np.empty_like(u)
    lib().oracle_stage(_p(u), _p(f), H, W, m, nk, centers.size, _p(kernels_t),
                       _p(weights_t), _p(centers), float(gamma), float(lam),
                       _p(out))
    return out


def force(u, kernels_t, weights_t, centers, gamma) -> np.ndarray:
    u = _c64(u)
    kernels_t = _c64(kernels_t); weights_t = _c64(weights_t)
    centers = _c64(centers)
    nk, m, _ = kernels_t.shape
    H, W = u.shape
    out = np.empty_like(u)
    lib().oracle_force(_p(u), H, W, m, nk, centers.size, _p(kernels_t),
                       _p(weights_t), _p(centers), float(gamma), _p(out))
    return out


def conv2d(img, k) -> np.ndarray:
    img = _c64(img); k = _c64(k)
    H, W = img.shape
    out = np.empty_like(img)
    lib().oracle_conv2d(_p(img), H, W, _p(k), k.shape[0], _p(out))
    return out


def prox_idiv(u_tilde, f, lam) -> np.ndarray:
    u_tilde = _c64(u_tilde); f = _c64(f)
    out = np.empty_like(u_tilde)
    lib().oracle_prox_idiv(_p(u_tilde), _p(f), float(lam), _p(out),
                           u_tilde.size)
    return out


def psnr(test, reference, peak: float) -> float:
    """metrics.py:28-39"""
    test = np.asarray(test, dtype=np.float64)
    reference = np.asarray(reference, dtype=np.float64)
    mse = float(np.mean((test - reference) ** 2))
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(peak * peak / mse)


def threads() -> int:
    return int(lib().oracle_max_threads())


def philox4x32_10(ctr, key) -> tuple:
    """Philox4x32-10 block (the GPU speckle generator's integer core)."""
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return tuple(o)


def speckle_field(shape, looks: int, seed: int, base: int = 0) -> np.ndarray:
    """float64 restatement of tnrd_sample_speckle's field sqrt(G/L) for the
    pixel indices base .. base + prod(shape) (see tnrd_oracle.c)."""
    out = np.empty(int(np.prod(shape)), dtype=np.float64)
    lib().oracle_speckle_field(_p(out), out.size, int(shape[-1]), int(looks), int(seed),
                               int(base))
    return out.reshape(shape)

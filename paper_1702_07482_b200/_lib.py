"""ctypes binding of the C ABI in include/tnrd.h (libtnrd.so, built in-tree).

There is no CPU fallback: if the CUDA library is missing or no GPU is
visible, every compute entry point raises.  Symbol-level loading works
without a GPU (tests check the exports on CPU).
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TNRD_LIB_PATH") or os.path.join(_HERE, "libtnrd.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "tnrd.h")

TNRD_OK = 0
TNRD_EINVAL = 1
TNRD_ENONFINITE = 2
TNRD_ECUDA = 3
TNRD_EUNSUPPORTED = 4

STAGE_FLOOR_INPUT = 0x1
STAGE_TOP_HALO = 0x2
STAGE_BOTTOM_HALO = 0x4
STAGE_FORCE = 0x8
STAGE_CHECK_F = 0x10
STAGE_PROJECTED = 0x20
VARIANT_PROX, VARIANT_PROJECTED = 0, 1

STATUS_WORDS = 2

_c_int = ctypes.c_int
_c_i64 = ctypes.c_int64
_c_u32 = ctypes.c_uint32
_c_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); the test suite checks this table against the
# declarations in include/tnrd.h.
SIGNATURES = {
    "tnrd_last_error": (ctypes.c_char_p, []),
    "tnrd_version": (ctypes.c_char_p, []),
    "tnrd_model_create": (_c_int, [_c_int, _c_int, _c_int, _c_int, _dp, _dp,
                                   _c_dbl, _c_dbl, _c_dbl, _dp, _c_int,
                                   ctypes.POINTER(_vp)]),
    "tnrd_model_destroy": (_c_int, [_vp]),
    "tnrd_model_set_variant": (_c_int, [_vp, _c_int, _c_dbl]),
    "tnrd_model_info": (_c_int, [_vp] + [ctypes.POINTER(_c_int)] * 5),
    "tnrd_model_rbf_fit_cubic": (_c_int, [_vp, ctypes.POINTER(_c_dbl), ctypes.POINTER(_c_dbl),
                                         ctypes.POINTER(_c_int)]),
    "tnrd_model_rbf_fit": (_c_int, [_vp, ctypes.POINTER(_c_dbl),
                                    ctypes.POINTER(_c_dbl),
                                    ctypes.POINTER(_c_dbl),
                                    ctypes.POINTER(_c_int)]),
    "tnrd_set_stage_kernel": (_c_int, [_c_int]),
    "tnrd_set_param_taps": (_c_int, [_c_int]),
    "tnrd_set_cluster_size": (_c_int, [_c_int]),
    "tnrd_set_zfield_passes": (_c_int, [_c_int]),
    "tnrd_status_reset": (_c_int, [_vp, _vp]),
    "tnrd_status_decode": (_c_int, [ctypes.POINTER(_c_u32),
                                    ctypes.POINTER(_c_int)]),
    "tnrd_stage": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _c_int, _c_int,
                            _c_int, _c_i64, _c_i64, _c_u32, _vp, _vp]),
    "tnrd_stage_force": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                  _c_int, _c_i64, _c_i64, _c_u32, _vp, _vp]),
    "tnrd_despeckle": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int,
                                _c_i64, _c_i64, _vp, _vp]),
    "tnrd_plan_create": (_c_int, [_vp, _c_int, _c_int, _c_int,
                                  ctypes.POINTER(_vp)]),
    "tnrd_plan_destroy": (_c_int, [_vp]),
    "tnrd_plan_despeckle_host": (_c_int, [_vp, _vp, _vp]),
    "tnrd_plan_despeckle_device": (_c_int, [_vp, _vp, _vp]),
    "tnrd_plan_despeckle_host_many": (_c_int, [_vp, _vp, _vp, _c_int, ctypes.POINTER(_c_int)]),
    "tnrd_plan_check": (_c_int, [_vp, ctypes.POINTER(_c_int)]),
    "tnrd_plan_stream": (_vp, [_vp]),
    "tnrd_plan_f_device": (_vp, [_vp]),
    "tnrd_plan_u_device": (_vp, [_vp]),
    "tnrd_conv2d": (_c_int, [_vp, _vp, _c_int, _c_int, _c_i64, _dp, _c_int,
                             _vp]),
    "tnrd_prox_idiv": (_c_int, [_vp, _vp, _vp, _c_i64, _c_dbl, _vp]),
    "tnrd_stage_backward": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                     ctypes.POINTER(_c_dbl), _dp, _dp, _vp]),
    "tnrd_conv2d_adjoint": (_c_int, [_vp, _vp, _c_int, _c_int, _dp, _c_int, _vp]),
    "tnrd_patch_correlation": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _dp, _vp]),
    "tnrd_sample_speckle": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _c_i64,
                                     _c_i64, _c_int, ctypes.c_uint64, _vp, _vp]),
    "tnrd_philox4x32_10": (None, [ctypes.POINTER(_c_u32), ctypes.POINTER(_c_u32),
                                  ctypes.POINTER(_c_u32)]),
    "tnrd_launch_count": (ctypes.c_uint64, []),
    "tnrd_build_features": (_c_u32, []),
    "tnrd_launch_count_reset": (None, []),
    "tnrd_probe": (_c_int, [_c_int, _c_int, _c_int, _vp,
                            ctypes.POINTER(ctypes.c_double)]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libtnrd.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA extension not built: {LIB_PATH} is missing "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        mode = os.environ.get("TNRD_STAGE_KERNEL")  # experiments: 0 auto, 1 cuda-core, 2 tcgen05
        if mode:
            L.tnrd_set_stage_kernel(int(mode))
        passes = os.environ.get("TNRD_ZF_PASSES")  # experiments: 3, 4 or 6
        if passes:
            L.tnrd_set_zfield_passes(int(passes))
    return _lib


def last_error() -> str:
    msg = load().tnrd_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map a C ABI return code onto the reference's exception types."""
    if rc == TNRD_OK:
        return
    msg = last_error()
    if rc == TNRD_EINVAL:
        raise ValueError(msg)
    if rc == TNRD_ENONFINITE:
        raise FloatingPointError(msg)
    if rc == TNRD_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg or f"tnrd error {rc}")


def dptr(a) -> _dp:
    return a.ctypes.data_as(_dp)


KERNEL_AUTO, KERNEL_CUDA_CORE, KERNEL_TENSOR_CORE = 0, 1, 2
KERNEL_SMALL_TILES, KERNEL_LARGE_TILES = 3, 4
KERNEL_TC_PHASED = 5
KERNEL_SPLIT_LARGE, KERNEL_SPLIT_SMALL = 6, 7
KERNEL_ZFIELD = 8
KERNEL_CLUSTER_LARGE, KERNEL_CLUSTER_SMALL = 10, 11
KERNEL_TC_ADJOINT = 12


def set_stage_kernel(mode: int) -> None:
    """0 auto, 1 CUDA-core, 2 tcgen05 forward GEMM, 3/4 CUDA-core tile
    kernel with small/large tiles forced, 6/7 split kernel, 10/11 cluster
    kernel, 12 tensor-core adjoint (include/tnrd.h)."""
    check(load().tnrd_set_stage_kernel(int(mode)))


def set_cluster_size(ctas: int) -> None:
    """CTAs per cluster of the cluster kernels (modes 10 / 11 and auto on
    small grids): 0 = from the grid size, 2..8 forced."""
    check(load().tnrd_set_cluster_size(int(ctas)))


def set_param_taps(on: bool) -> None:
    """Large-tile CUDA-core kernels: taps from the kernel parameter space
    (True, default) or staged in shared memory (False); same bits."""
    check(load().tnrd_set_param_taps(int(bool(on))))


FEATURE_EXPERIMENTS = 0x1


def has_experiments() -> bool:
    """True if the opt-in tensor-core / dataflow kernels are compiled in
    (-DTNRD_EXPERIMENTS, tools/build_experiments.sh)."""
    return bool(load().tnrd_build_features() & FEATURE_EXPERIMENTS)


def launch_count() -> int:
    return int(load().tnrd_launch_count())


def launch_count_reset() -> None:
    load().tnrd_launch_count_reset()

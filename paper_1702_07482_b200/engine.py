"""Device-side engine: one uploaded model, stream-ordered launches, plans.

This is the layer between the reference-shaped Python API (diffusion.py)
and the C ABI (include/tnrd.h).  PyTorch is used only for device memory,
streams and torch.distributed plumbing; every kernel that touches the data
is in libtnrd.so.
"""
from __future__ import annotations

import ctypes
import hashlib
import math
import threading
from typing import Sequence

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda() -> None:
    if not torch().cuda.is_available():
        raise RuntimeError("no CUDA device is visible: the TNRD path is GPU-only "
                           "(there is no CPU fallback)")


def _stream_handle(stream=None) -> ctypes.c_void_p:
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def stream_ctx(stream=None):
    """Make ``stream`` current for the duration of a call: temporaries are
    then allocated on the stream their kernels run on (the caching
    allocator reuses a freed block only in that stream's order) and a status
    read (.cpu()) is ordered after those kernels."""
    import contextlib
    return contextlib.nullcontext() if stream is None else torch().cuda.stream(stream)


def _ptr(tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(tensor.data_ptr())


def rbf_grid_params(count: int, radius: float, bandwidth=None):
    """(mu0, delta, gamma) of RbfGrid (influence.py:29-37): centres are
    np.linspace(-radius, radius, count), gamma defaults to the spacing."""
    delta = 2.0 * radius / (count - 1)
    gamma = float(bandwidth) if bandwidth is not None else delta
    return -float(radius), float(delta), float(gamma)


def params_fingerprint(m: int, kernels: np.ndarray, weights: np.ndarray,
                       lams: np.ndarray, grid: tuple) -> str:
    h = hashlib.blake2b(digest_size=16)
    h.update(np.asarray([m], dtype=np.int64).tobytes())
    for a in (kernels, weights, lams, np.asarray(grid, dtype=np.float64)):
        a = np.ascontiguousarray(a, dtype=np.float64)
        h.update(np.asarray(a.shape, dtype=np.int64).tobytes())
        h.update(a.tobytes())
    return h.hexdigest()


class Status:
    """Device status block (2 x uint32): first non-finite stage, f flags."""

    def __init__(self, device):
        t = torch()
        self.buf = t.empty(_lib.STATUS_WORDS, dtype=t.int32, device=device)

    def reset(self, stream=None) -> None:
        _lib.check(_lib.load().tnrd_status_reset(_ptr(self.buf),
                                                 _stream_handle(stream)))

    def check(self) -> None:
        """Synchronise (via the D2H copy) and raise the reference's error."""
        host = self.buf.cpu().numpy().view(np.uint32).copy()
        arr = (ctypes.c_uint32 * _lib.STATUS_WORDS)(*host.tolist())
        bad = ctypes.c_int(-1)
        _lib.check(_lib.load().tnrd_status_decode(arr, ctypes.byref(bad)))


class DeviceModel:
    """A DiffusionModel uploaded to one GPU (tnrd_model_create).

    kernels: (T, nk, m, m) float64 -- the reference's true-convolution
    kernels k_i = coeffs @ basis.T (diffusion.py:76-77); weights (T, nk, M);
    lams (T,) with lambda = exp(beta) (diffusion.py:72-74).
    """

    def __init__(self, kernels, weights, lams, grid, device=None, variant: int = 0,
                 floor: float = 1.0):
        require_cuda()
        t = torch()
        L = _lib.load()
        k = np.ascontiguousarray(kernels, dtype=np.float64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        lm = np.ascontiguousarray(lams, dtype=np.float64)
        if k.ndim != 4 or k.shape[2] != k.shape[3]:
            raise ValueError("kernels must be (T, nk, m, m)")
        T, nk, m, _ = k.shape
        if w.ndim != 3 or w.shape[:2] != (T, nk):
            raise ValueError("weights must be (T, nk, M)")
        if lm.shape != (T,):
            raise ValueError("need one lambda per stage")
        M = w.shape[2]
        mu0, delta, gamma = grid
        self.device = t.device("cuda", t.cuda.current_device()
                               if device is None else int(device))
        self.m, self.nk, self.T, self.M = m, nk, T, M
        self.grid = (mu0, delta, gamma)
        h = ctypes.c_void_p()
        _lib.check(L.tnrd_model_create(m, nk, T, M, _lib.dptr(k), _lib.dptr(w),
                                       mu0, delta, gamma, _lib.dptr(lm),
                                       self.device.index, ctypes.byref(h)))
        self.handle = h
        self.variant, self.floor = int(variant), float(floor)
        if self.variant != _lib.VARIANT_PROX:
            _lib.check(L.tnrd_model_set_variant(h, self.variant, self.floor))
        fast = ctypes.c_int(0)
        _lib.check(L.tnrd_model_info(h, None, None, None, None,
                                     ctypes.byref(fast)))
        self.fast_rbf = bool(fast.value)
        err, e32 = ctypes.c_double(0), ctypes.c_double(0)
        scale, ni = ctypes.c_double(0), ctypes.c_int(0)
        _lib.check(L.tnrd_model_rbf_fit(h, ctypes.byref(err), ctypes.byref(e32),
                                        ctypes.byref(scale), ctypes.byref(ni)))
        # polynomial RBF tables: (max |p - phi| float64 coeffs, fp32 coeffs,
        # max sum|w|, intervals)
        self.rbf_fit = (err.value, e32.value, scale.value, ni.value)
        # cubic table of the parameter-space-taps kernels: (max |p - phi|
        # float64 coeffs, fp32 coeffs, intervals; 0 = none)
        _lib.check(L.tnrd_model_rbf_fit_cubic(h, ctypes.byref(err), ctypes.byref(e32),
                                              ctypes.byref(ni)))
        self.rbf_fit_cubic = (err.value, e32.value, ni.value)
        self._plans = {}
        self._plan_lock = threading.Lock()
        self._status = {}

    # ---------------------------------------------------------- lifecycle
    def close(self) -> None:
        L = _lib._lib
        if L is None or self.handle is None:
            return
        for p in self._plans.values():
            L.tnrd_plan_destroy(p)
        self._plans.clear()
        L.tnrd_model_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def radius(self) -> int:
        return self.m // 2

    def status(self) -> Status:
        # one status block per (thread, current stream): calls on different
        # streams never share one
        key = (threading.get_ident(), torch().cuda.current_stream(self.device).cuda_stream)
        s = self._status.get(key)
        if s is None:
            s = self._status[key] = Status(self.device)
        return s

    # ---------------------------------------------------------- device API
    def _shape(self, x):
        if x.dim() == 2:
            return 1, x.shape[0], x.shape[1]
        if x.dim() == 3:
            return x.shape[0], x.shape[1], x.shape[2]
        raise ValueError(f"expected (H, W) or (B, H, W), got {tuple(x.shape)}")

    def _check_tensor(self, x, name):
        t = torch()
        if x.device != self.device:
            raise ValueError(f"{name} is on {x.device}, model on {self.device}")
        if x.dtype != t.float32:
            raise ValueError(f"{name} must be float32")
        if x.stride(-1) != 1:
            raise ValueError(f"{name} rows must be contiguous")

    def despeckle(self, f, out=None, work=None, stream=None, check=True):
        """run_diffusion on device tensors: f (H, W) or (B, H, W) fp32 CUDA.
        Returns u_T (same shape).  With check=False the status block is left
        for a later ``status().check()`` on the same stream (no host
        synchronisation).  ``stream``: run (and allocate temporaries) there."""
        with stream_ctx(stream):
            return self._despeckle(f, out, work, check)

    def _despeckle(self, f, out, work, check):
        t = torch()
        self._check_tensor(f, "f")
        B, H, W = self._shape(f)
        if out is None:
            out = t.empty_like(f, memory_format=t.contiguous_format)
        if work is None and self.T > 1:
            work = t.empty_like(out)
        for name, x in (("out", out), ("work", work)):
            if x is not None:
                self._check_tensor(x, name)
                if x.shape != f.shape or x.stride() != out.stride():
                    raise ValueError(f"{name} must match f's shape and out's strides")
        if f.stride() != out.stride():
            # the kernels take ONE row / image stride for f, out and work
            f2 = t.empty_strided(out.shape, out.stride(), dtype=f.dtype, device=f.device)
            f2.copy_(f)
            f = f2
        assert f.stride() == out.stride() and (work is None or work.stride() == out.stride())
        ld = out.stride(-2)
        img_stride = out.stride(0) if out.dim() == 3 else ld * H
        st = self.status()
        st.reset()
        _lib.check(_lib.load().tnrd_despeckle(
            self.handle, _ptr(f), _ptr(out),
            _ptr(work) if work is not None else None, B, H, W, ld, img_stride,
            _ptr(st.buf), _stream_handle()))
        if check:
            st.check()
        return out

    def stage(self, t_index: int, u, f, out=None, flags: int = 0,
              stream=None, status: Status | None = None, rows=None):
        """One stage on device tensors.  ``rows`` = (row0, H) restricts the
        stage to rows [row0, row0 + H) of u/f/out (row strips: u must then
        carry the halo rows around that window when TOP/BOTTOM_HALO is set)."""
        with stream_ctx(stream):
            return self._stage(t_index, u, f, out, flags, status, rows)

    def stage_force(self, t_index: int, u, f, stream=None):
        """One stage returning (u_next, force) from ONE launch
        (tnrd_stage_force): diffusion_step's output and the force behind its
        trace's u~ = u - force."""
        with stream_ctx(stream):
            force = torch().empty_like(u)
            return self._stage(t_index, u, f, None, 0, None, None, force_out=force), force

    def _stage(self, t_index, u, f, out, flags, status, rows, force_out=None):
        t = torch()
        self._check_tensor(u, "u")
        self._check_tensor(f, "f")
        if out is None:
            out = t.empty_like(u)
        self._check_tensor(out, "out")
        B, H, W = self._shape(u)
        if u.stride() != f.stride() or u.stride() != out.stride():
            raise ValueError("u, f and out must share strides")
        ld = u.stride(-2)
        img_stride = u.stride(0) if u.dim() == 3 else ld * H
        row0 = 0
        if rows is not None:
            row0, H = int(rows[0]), int(rows[1])
        off = row0 * ld * u.element_size()
        st = status if status is not None else self.status()
        if status is None:
            st.reset()
        if force_out is not None:
            self._check_tensor(force_out, "force_out")
            if force_out.stride() != out.stride():
                raise ValueError("force_out must share out's strides")
            _lib.check(_lib.load().tnrd_stage_force(
                self.handle, int(t_index), ctypes.c_void_p(u.data_ptr() + off),
                ctypes.c_void_p(f.data_ptr() + off), ctypes.c_void_p(out.data_ptr() + off),
                ctypes.c_void_p(force_out.data_ptr() + off), B, H, W, ld, img_stride,
                int(flags), _ptr(st.buf), _stream_handle()))
        else:
            _lib.check(_lib.load().tnrd_stage(
                self.handle, int(t_index), ctypes.c_void_p(u.data_ptr() + off),
                ctypes.c_void_p(f.data_ptr() + off),
                ctypes.c_void_p(out.data_ptr() + off), B, H, W, ld, img_stride,
                int(flags), _ptr(st.buf), _stream_handle()))
        if status is None:
            st.check()
        return out

    # ---------------------------------------------------------- host API
    def _plan(self, B, H, W):
        key = (threading.get_ident(), B, H, W)
        p = self._plans.get(key)
        if p is None:
            with self._plan_lock:
                p = self._plans.get(key)
                if p is None:
                    h = ctypes.c_void_p()
                    _lib.check(_lib.load().tnrd_plan_create(
                        self.handle, B, H, W, ctypes.byref(h)))
                    p = self._plans[key] = h
        return p

    def despeckle_host_many(self, f: np.ndarray, out: np.ndarray | None = None):
        """Despeckle a sequence of HOST images f[i] ((count, H, W) or
        (count, B, H, W), fp32) through tnrd_plan_despeckle_host_many: the
        copies of one image overlap the stages of the next (pass pinned
        arrays, e.g. torch pin_memory().numpy(), for the overlap).  Raises
        the first failing image's error."""
        f = np.asarray(f, dtype=np.float32)
        if f.ndim == 3:
            count, B, (H, W) = f.shape[0], 1, f.shape[1:]
        elif f.ndim == 4:
            count, B, H, W = f.shape
        else:
            raise ValueError(f"expected (count, H, W) or (count, B, H, W), got {f.shape}")
        if not f.flags.c_contiguous:
            f = np.ascontiguousarray(f)
        if out is None:
            out = np.empty_like(f)
        elif out.shape != f.shape or out.dtype != np.float32 or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32 array like f")
        p = self._plan(B, H, W)
        bad = ctypes.c_int(-1)
        _lib.check(_lib.load().tnrd_plan_despeckle_host_many(
            p, f.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p),
            count, ctypes.byref(bad)))
        return out

    def despeckle_host(self, f: np.ndarray, out: np.ndarray | None = None):
        """Full despeckle of HOST fp32 arrays through the plan C ABI
        (tnrd_plan_despeckle_host: H2D, T stages, D2H, status check)."""
        f = np.ascontiguousarray(f, dtype=np.float32)
        if f.ndim == 2:
            B, (H, W) = 1, f.shape
        elif f.ndim == 3:
            B, H, W = f.shape
        else:
            raise ValueError(f"expected (H, W) or (B, H, W), got {f.shape}")
        if out is None:
            out = np.empty_like(f)
        elif out.shape != f.shape or out.dtype != np.float32 or \
                not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32 array like f")
        p = self._plan(B, H, W)
        _lib.check(_lib.load().tnrd_plan_despeckle_host(
            p, f.ctypes.data_as(ctypes.c_void_p),
            out.ctypes.data_as(ctypes.c_void_p)))
        return out


def model_kernels(model, stages: Sequence | None = None) -> np.ndarray:
    """(T, nk, m, m) float64 kernels of a DiffusionModel, exactly as the
    reference builds them (diffusion.py:76-77, 189)."""
    stages = model.stages if stages is None else stages
    return np.stack([s.kernels(model.basis, model.filter_size) for s in stages])


_CACHE: "dict[tuple, DeviceModel]" = {}
_CACHE_MAX = 16
_CACHE_LOCK = threading.Lock()


def cached_device_model(kernels, weights, lams, grid, variant: int = 0,
                        floor: float = 1.0) -> DeviceModel:
    """DeviceModel for explicit float64 parameter arrays, cached process-wide
    by (device, fingerprint of every parameter) so in-place edits of
    StageParams (as the reference's tests do) are seen and unchanged models
    are uploaded once."""
    require_cuda()
    kernels = np.ascontiguousarray(kernels, dtype=np.float64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    lams = np.ascontiguousarray(lams, dtype=np.float64)
    dev = torch().cuda.current_device()
    key = (dev, int(variant), float(floor),
           params_fingerprint(kernels.shape[-1], kernels, weights, lams, grid))
    with _CACHE_LOCK:
        dm = _CACHE.pop(key, None)
        if dm is None:
            while len(_CACHE) >= _CACHE_MAX:
                _CACHE.pop(next(iter(_CACHE)))  # freed by __del__ once unreferenced
            dm = DeviceModel(kernels, weights, lams, grid, device=dev, variant=variant,
                             floor=floor)
        _CACHE[key] = dm  # most recently used last
    return dm


def device_model_for(model, stages: Sequence | None = None,
                     kernels: np.ndarray | None = None) -> DeviceModel:
    """Cached DeviceModel for ``model`` (or for the given stage list /
    explicit (T, nk, m, m) kernels), see cached_device_model."""
    stages = list(model.stages if stages is None else stages)
    k = model_kernels(model, stages) if kernels is None else kernels
    w = np.stack([np.asarray(s.weights, dtype=np.float64) for s in stages])
    lams = np.array([math.exp(float(s.beta)) for s in stages])
    g = model.rbf
    projected = getattr(model, "variant", "prox") == "projected"
    return cached_device_model(k, w, lams, rbf_grid_params(g.count, g.radius, g.bandwidth),
                               variant=_lib.VARIANT_PROJECTED if projected else _lib.VARIANT_PROX,
                               floor=float(getattr(model, "floor", 1.0)))

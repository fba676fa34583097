"""Image validation and the mirror-padded convolution (drop-in for
specklediff.imageops, reference imageops.py:17-72).

``conv2d`` runs on the GPU (tnrd_conv2d); validation and error messages
follow the reference so callers see the same exceptions.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .engine import require_cuda, torch, _stream_handle, _ptr

# kept for API compatibility: the reference switches to FFT for m >= 9
# (imageops.py:14); the GPU path is always direct
FFT_KERNEL_CUTOFF = 9


def as_image(a, name: str = "image") -> np.ndarray:
    """imageops.py:17-26 -- finite 2D float64 array or ValueError."""
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2D, got shape {arr.shape}")
    if min(arr.shape) < 1:
        raise ValueError(f"{name} must have at least one pixel")
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains non-finite values")
    return arr


def as_kernel(k, name: str = "kernel") -> np.ndarray:
    """imageops.py:29-37 -- square, odd, finite."""
    arr = np.asarray(k, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise ValueError(f"{name} must be square 2D, got shape {arr.shape}")
    if arr.shape[0] % 2 == 0:
        raise ValueError(f"{name} side must be odd, got {arr.shape[0]}")
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains non-finite values")
    return arr


def check_fits(shape, m: int) -> None:
    """imageops.py:40-45 -- one mirror fold must suffice."""
    if m > 2 * min(shape) + 1:
        raise ValueError(
            f"kernel size {m} degenerate for image of shape {tuple(shape)}")


def rotate180(k) -> np.ndarray:
    """imageops.py:48-50 -- point reflection of a kernel."""
    return np.flip(as_kernel(k)).copy()


def conv2d(img, k, method: str = "auto") -> np.ndarray:
    """Same-size true convolution over a half-sample-symmetric padded image
    (imageops.py:53-72), computed on the GPU in fp32; returns float64."""
    img = as_image(img)
    k = as_kernel(k)
    check_fits(img.shape, k.shape[0])
    if method not in ("auto", "direct", "fft"):
        raise ValueError(f"unknown convolution method {method!r}")
    require_cuda()
    t = torch()
    H, W = img.shape
    x = t.from_numpy(img.astype(np.float32)).cuda()
    out = t.empty_like(x)
    kk = np.ascontiguousarray(k)
    _lib.check(_lib.load().tnrd_conv2d(_ptr(x), _ptr(out), H, W, W,
                                       _lib.dptr(kk), k.shape[0],
                                       _stream_handle()))
    return out.cpu().numpy().astype(np.float64)


def conv2d_adjoint(img, k, method: str = "auto") -> np.ndarray:
    """Exact transpose of ``conv2d(., k)`` (imageops.py:90-106): satisfies
    <conv2d(a, k), b> == <a, conv2d_adjoint(b, k)>.  GPU, fp32 (the mirror
    padding's adjoint is folded per output pixel); returns float64."""
    img = as_image(img)
    k = as_kernel(k)
    check_fits(img.shape, k.shape[0])
    if method not in ("auto", "direct", "fft"):
        raise ValueError(f"unknown convolution method {method!r}")
    require_cuda()
    t = torch()
    H, W = img.shape
    x = t.from_numpy(img.astype(np.float32)).cuda()
    out = t.empty_like(x)
    kk = np.ascontiguousarray(k)
    _lib.check(_lib.load().tnrd_conv2d_adjoint(_ptr(x), _ptr(out), H, W, _lib.dptr(kk),
                                               k.shape[0], _stream_handle()))
    return out.cpu().numpy().astype(np.float64)


def patch_correlation(base, adj, m: int) -> np.ndarray:
    """C[a, b] = sum_p pad(base)[p + (a, b)] adj[p] with pad = symmetric
    padding by m // 2 (imageops.py:109-127); rotate180(C) is the gradient of
    <adj, conv2d(base, k)> w.r.t. k.  GPU, fp32 products, float64 sums."""
    base = as_image(base, "base")
    adj = as_image(adj, "adj")
    if base.shape != adj.shape:
        raise ValueError("base and adj must share dimensions")
    if m < 1 or m % 2 != 1:
        raise ValueError(f"kernel side must be odd, got {m}")
    check_fits(base.shape, m)
    require_cuda()
    t = torch()
    H, W = base.shape
    b = t.from_numpy(base.astype(np.float32)).cuda()
    a = t.from_numpy(adj.astype(np.float32)).cuda()
    out = np.empty((m, m), dtype=np.float64)
    _lib.check(_lib.load().tnrd_patch_correlation(_ptr(b), _ptr(a), H, W, m, _lib.dptr(out),
                                                  _stream_handle()))
    return out

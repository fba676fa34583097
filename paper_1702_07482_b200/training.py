"""Gradients of the unrolled diffusion on the GPU.

Drop-in for the gradient path of the reference's ``specklediff.training``
(training.py:31-166): ``loss``, ``loss_grad``, ``StageGradients``,
``backprop_adjoint``, ``grad_stage_params`` and ``loss_and_gradients`` with
the reference's signatures.  Each stage's backward (training.py:69-123
``_stage_backward``) runs as CUDA kernels through ``tnrd_stage_backward``
(csrc/tnrd_train.cuh): z / phi / phi' are recomputed on the GPU from u_prev
instead of being stored as traces (the fused forward never materialises
them), the parameter gradients are fixed-order float64 reductions, and the
host maps the kernel-space gradient to basis coefficients exactly like
training.py:110.  Arithmetic is fp32 on the device; gradients agree with the
float64 reference to ~1e-5 relative (tests/test_gpu_training.py).

The optimiser loop (L-BFGS-B schedules, training.py:170-454) stays out of
scope: it is host-side scipy driving these gradients.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .diffusion import initial_state
from .engine import _ptr, _stream_handle, device_model_for, require_cuda, torch
from .imageops import as_image


def loss(u_out, u_gt) -> float:
    """Quadratic training loss 0.5 ||u_out - u_gt||^2 (training.py:31-38)."""
    u_out = as_image(u_out, "u_out")
    u_gt = as_image(u_gt, "u_gt")
    if u_out.shape != u_gt.shape:
        raise ValueError("loss operands must share dimensions")
    d = u_out - u_gt
    return 0.5 * float(np.dot(d.ravel(), d.ravel()))


def loss_grad(u_out, u_gt) -> np.ndarray:
    """training.py:41-42"""
    return np.asarray(u_out, float) - np.asarray(u_gt, float)


@dataclass
class StageGradients:
    """training.py:45-49"""
    beta: float
    coeffs: np.ndarray
    weights: np.ndarray


def _dev(a: np.ndarray):
    return torch().from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def stage_backward_device(dm, t: int, u_prev, f, g_next, basis: np.ndarray | None = None,
                          want_params: bool = True, want_adjoint: bool = True, stream=None):
    """One stage backward on device tensors (dense (H, W) fp32 CUDA):
    returns (g_prev tensor or None, StageGradients or None).  ``basis`` maps
    the kernel-space gradient to coefficients (training.py:110)."""
    t_ = torch()
    H, W = u_prev.shape
    g_prev = t_.empty_like(u_prev) if want_adjoint else None
    beta = ctypes.c_double(0.0)
    gk = gw = None
    if want_params:
        gk = np.empty((dm.nk, dm.m * dm.m), dtype=np.float64)
        gw = np.empty((dm.nk, dm.M), dtype=np.float64)
    _lib.check(_lib.load().tnrd_stage_backward(
        dm.handle, int(t), _ptr(u_prev), _ptr(f),
        _ptr(g_next) if g_next is not None else None,
        _ptr(g_prev) if g_prev is not None else None, H, W,
        ctypes.byref(beta) if want_params else None,
        gk.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if want_params else None,
        gw.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if want_params else None,
        _stream_handle(stream)))
    grads = None
    if want_params:
        coeffs = gk @ basis if basis is not None else gk   # (nk, m^2) @ (m^2, m^2-1)
        grads = StageGradients(float(beta.value), coeffs, gw)
    return g_prev, grads


def _stage_backward(trace, stage, f, g_next, model, want_params=True, want_adjoint=True):
    require_cuda()
    f = as_image(f, "f")
    dm = device_model_for(model, stages=[stage])
    u = _dev(as_image(trace.u_prev, "u_prev"))
    g_prev, grads = stage_backward_device(
        dm, 0, u, _dev(f), _dev(as_image(g_next, "adjoint")), model.basis,
        want_params, want_adjoint)
    g = g_prev.cpu().numpy().astype(np.float64) if g_prev is not None else None
    return g, grads


def backprop_adjoint(trace, stage, f, adjoint_next, model) -> np.ndarray:
    """(d u_next / d u_prev)^T adjoint_next (training.py:52-57); only
    trace.u_prev is read (z / phi are recomputed on the GPU)."""
    g_prev, _ = _stage_backward(trace, stage, f, adjoint_next, model, want_params=False)
    return g_prev


def grad_stage_params(trace, stage, f, adjoint_next, model) -> StageGradients:
    """Gradients w.r.t. one stage's {beta, coeffs, weights}
    (training.py:60-66)."""
    _, grads = _stage_backward(trace, stage, f, adjoint_next, model, want_adjoint=False)
    return grads


def _forward_device(dm, f_dev, upto: int, u0: np.ndarray | None, model):
    """u_0 .. u_{upto+1} on the device (training.py:126-137 without traces)."""
    u = _dev(initial_state(f_dev.cpu().numpy().astype(np.float64), model) if u0 is None
             else np.asarray(u0, dtype=np.float64))
    us = [u]
    for t in range(upto + 1):
        u = dm.stage(t, u, f_dev)      # raises FloatingPointError like the reference
        us.append(u)
    return us


def loss_and_gradients(model, pairs, grad_stages, loss_stage: int, inputs=None):
    """Total loss at the output of ``loss_stage`` plus gradients for the
    requested stages, accumulated over samples in ascending order
    (training.py:140-166)."""
    require_cuda()
    grad_stages = sorted(grad_stages)
    lowest = grad_stages[0]
    dm = device_model_for(model)
    basis = model.basis
    total = 0.0
    acc = {t: None for t in grad_stages}
    for s, pair in enumerate(pairs):
        f = as_image(pair.noisy, "f")
        f_dev = _dev(f)
        u0 = None if inputs is None else inputs[s]
        us = _forward_device(dm, f_dev, loss_stage, u0, model)
        u_out = us[loss_stage + 1].cpu().numpy().astype(np.float64)
        total += loss(u_out, pair.clean)
        g = _dev(loss_grad(u_out, pair.clean))
        for t in range(loss_stage, lowest - 1, -1):
            g_prev, grads = stage_backward_device(
                dm, t, us[t], f_dev, g, basis, want_params=t in acc,
                want_adjoint=t > lowest)
            if t in acc:
                if acc[t] is None:
                    acc[t] = grads
                else:
                    acc[t].beta += grads.beta
                    acc[t].coeffs += grads.coeffs
                    acc[t].weights += grads.weights
            g = g_prev
    return total, acc

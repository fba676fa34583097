"""CPU numerical model of the stage arithmetic under different schemes, to
decide BEFORE building a kernel whether a tensor-core formulation can meet
the 1e-4 relative bar on the hardest golden case (zeros_in_f).

Schemes for the forward filter bank / the adjoint:
  ffma       direct 49-tap fp32 FMA chains (the CUDA-core kernels)
  tc_direct  forward as a 3-piece tf32 tensor-core GEMM over the taps (the
             z-field kernel); adjoint ffma
  dct        separable DCT basis: t_pq = conv(u, a_p x a_q) by fp32 FMA
             (column then row pass), z = C t as a 3xTF32 tensor-core GEMM
             over the m^2-1 basis atoms; adjoint psi = C^T phi on the tensor
             cores, force = sum_pq corr(psi_pq, a_p x a_q) separably in fp32

Tensor-core accumulation model: products of tf32 operands exact; per MMA
(K = 8) the accumulator and the 8 products are aligned to the largest
exponent and truncated to F fraction bits, summed, and the result is
truncated to fp32.  F is calibrated against the z-field kernel's measured
max relative error on zeros_in_f (1.94e-4).
Test/analysis tool only."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from conftest import golden_model, load_golden, parity_stats  # noqa: E402
import paper_1702_07482_b200 as tn  # noqa: E402

F_BITS = int(os.environ.get("TC_FBITS", "23"))


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def fma32(a, b, c):
    return f32(a * b + c)


def trunc_bits(x, bits):
    m, e = np.frexp(x)
    return np.ldexp(np.trunc(m * 2.0 ** bits), e - bits)


def tf32(x):
    m, e = np.frexp(x)
    return np.ldexp(np.round(m * 2.0 ** 11), e - 11)


def mma(acc, prods):
    """acc (...), prods (..., 8) exact -> acc' per the truncation model"""
    terms = np.concatenate([acc[..., None], prods], axis=-1)
    mx = np.max(np.abs(terms), axis=-1)
    _, emax = np.frexp(np.where(mx > 0, mx, 1.0))
    q = np.ldexp(1.0, emax - F_BITS)[..., None]
    s = np.sum(np.trunc(terms / q) * q, axis=-1)
    return trunc_bits(s, 24)


def pad(x, r):
    return np.pad(x, r, mode="symmetric")


def split3(x):
    h0 = tf32(x)
    r1 = f32(x - h0)
    h1 = tf32(r1)
    h2 = tf32(f32(r1 - h1))
    return [h0, h1, h2]


def forward_ffma(u, k):
    m = k.shape[0]
    r = m // 2
    H, W = u.shape
    up = pad(u, r)
    z = np.zeros((H, W))
    for a in range(m):
        for b in range(m):
            z = fma32(f32(k[m - 1 - a, m - 1 - b]), up[a:a + H, b:b + W], z)
    return z


def forward_tc_direct(u, k):
    m = k.shape[0]
    r = m // 2
    H, W = u.shape
    up = pad(u, r)
    upc = split3(up)
    kc = split3(f32(k))
    passes = [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)]
    z = np.zeros((H, W))
    for a in range(m):
        for (pu, pk) in passes:
            prods = np.zeros((H, W, 8))
            for b in range(m):
                prods[..., b] = kc[pk][m - 1 - a, m - 1 - b] * upc[pu][a:a + H, b:b + W]
            z = mma(z, prods)
    return z


def atoms(m):
    n = np.arange(m)
    A = np.empty((m, m))
    A[0] = np.sqrt(1.0 / m)
    for p in range(1, m):
        A[p] = np.sqrt(2.0 / m) * np.cos(np.pi * (n + 0.5) * p / m)
    return A


def gemm_tc(X, Bm, order):
    """X (P, K) fp32 rows, Bm (K, N) fp32: 3xTF32 tensor-core GEMM, K-steps
    of 8, passes in `order` per K-step"""
    P, K = X.shape
    N = Bm.shape[1]
    Kp = (K + 7) // 8 * 8
    Xp = np.zeros((P, Kp)); Xp[:, :K] = X
    Bp = np.zeros((Kp, N)); Bp[:K] = Bm
    xh = tf32(Xp); xl = tf32(f32(Xp - xh))
    bh = tf32(Bp); bl = tf32(f32(Bp - bh))
    pieces = {"hh": (xh, bh), "lh": (xl, bh), "hl": (xh, bl)}
    D = np.zeros((P, N))
    if order == "split":           # passes accumulated separately, summed in fp32
        outs = []
        for name in ("lh", "hl", "hh"):
            Dp = np.zeros((P, N))
            xa, ba = pieces[name]
            for ks in range(Kp // 8):
                prods = xa[:, None, 8 * ks:8 * ks + 8] * ba[8 * ks:8 * ks + 8].T[None]
                Dp = mma(Dp, prods)
            outs.append(Dp)
        return f32(f32(outs[0] + outs[1]) + outs[2])
    for ks in range(Kp // 8):
        for name in order:
            xa, ba = pieces[name]
            prods = xa[:, None, 8 * ks:8 * ks + 8] * ba[8 * ks:8 * ks + 8].T[None]
            D = mma(D, prods)
    return D


def forward_dct(u, C, A, order):
    """t_pq by separable fp32 FMA (column pass then row pass, true conv),
    z = C t on the tensor cores"""
    m = A.shape[0]
    r = m // 2
    H, W = u.shape
    up = pad(u, r)
    A32 = f32(A)
    ts = []
    for p in range(m):
        w = np.zeros((H, W + 2 * r))
        for a in range(m):           # true conv: u[y + r - a] * A_p[a]
            w = fma32(A32[p, a], up[2 * r - a:2 * r - a + H, :], w)
        for q in range(m):
            if p == 0 and q == 0:
                continue
            t = np.zeros((H, W))
            for b in range(m):
                t = fma32(A32[q, b], w[:, 2 * r - b:2 * r - b + W], t)
            ts.append(t)
    T = np.stack(ts, axis=-1).reshape(H * W, -1)
    Z = gemm_tc(T, f32(C).T, order)        # (HW, nk)
    return Z.reshape(H, W, -1)


def backward_dct(phi, C, A, order):
    """psi = C^T phi (tensor cores), force = sum_pq corr(psi_pq, a_p x a_q),
    x pass then y pass in fp32"""
    H, W, nk = phi.shape
    m = A.shape[0]
    r = m // 2
    A32 = f32(A)
    Psi = gemm_tc(phi.reshape(H * W, nk), f32(C), order).reshape(H, W, -1)
    force = np.zeros((H, W))
    hp = []
    k = 0
    for p in range(m):
        h = np.zeros((H, W))
        for q in range(m):
            if p == 0 and q == 0:
                continue
            pp = pad(Psi[..., k], r)[r:r + H, :]    # mirror in x only
            k += 1
            for b in range(m):                      # correlation: psi[x + b - r]
                h = fma32(A32[q, b], pp[:, b:b + W], h)
        hp.append(h)
    for p in range(m):
        hpad = pad(hp[p], r)[:, r:r + W]
        for a in range(m):
            force = fma32(A32[p, a], hpad[a:a + H, :], force)
    return force


def backward_ffma(phi, kernels):
    H, W, nk = phi.shape
    m = kernels.shape[1]
    r = m // 2
    force = np.zeros((H, W))
    for i in range(nk):
        pp = pad(phi[..., i], r)
        for a in range(m):
            for b in range(m):
                force = fma32(f32(kernels[i, a, b]), pp[a:a + H, b:b + W], force)
    return force


def rbf(z, w, mu, gamma):
    G = np.exp(-(z[..., None] - mu) ** 2 / (2 * gamma ** 2))
    return f32(G @ w)


def prox32(u, force, f, lam):
    a = 1 + 2 * lam
    ff = np.maximum(f32(f), 1e-6)
    ut = f32(u - force)
    fl2 = f32(ff * ff)
    root = f32(np.sqrt(f32(ut * ut + f32(8 * a * lam) * fl2)))
    pos = f32(f32(ut + root) * f32(1 / (2 * a)))
    neg = f32(f32(f32(4 * lam) * fl2) / f32(root - ut))
    return np.where(ut >= 0, pos, neg)


def run(name, fwd, bwd, order=("lh", "hl", "hh")):
    g = load_golden(name)
    model = golden_model(g)
    m = model.filter_size
    basis = tn.zero_mean_basis(m)
    A = atoms(m)
    grid = model.rbf
    mu = np.linspace(-grid.radius, grid.radius, grid.count)
    gamma = grid.bandwidth if grid.bandwidth else 2 * grid.radius / (grid.count - 1)
    f = f32(g["f"])
    u = np.maximum(f, 1e-6)
    for st in model.stages:
        K = st.kernels(basis, m)
        C = st.coeffs
        w = st.weights
        if fwd == "ffma":
            z = np.stack([forward_ffma(u, K[i]) for i in range(K.shape[0])], -1)
        elif fwd == "tc_direct":
            z = np.stack([forward_tc_direct(u, K[i]) for i in range(K.shape[0])], -1)
        else:
            z = forward_dct(u, C, A, order)
        phi = np.stack([rbf(z[..., i], w[i], mu, gamma) for i in range(K.shape[0])], -1)
        force = backward_ffma(phi, K) if bwd == "ffma" else backward_dct(phi, C, A, order)
        u = prox32(u, force, f, st.lam)
    return parity_stats(u, g["u"])


if __name__ == "__main__":
    names = sys.argv[1:] or ["zeros_in_f"]
    for name in names:
        for fwd, bwd, order in [("ffma", "ffma", None), ("tc_direct", "ffma", None),
                                ("dct", "dct", ("lh", "hl", "hh")),
                                ("dct", "dct", ("hh", "lh", "hl")),
                                ("dct", "dct", "split"),
                                ("dct", "ffma", ("lh", "hl", "hh")),
                                ("ffma", "dct", ("lh", "hl", "hh"))]:
            st = run(name, fwd, bwd, order) if order else run(name, fwd, bwd)
            print(f"F={F_BITS} {name:12s} fwd={fwd:9s} bwd={bwd:5s} order={order}: "
                  f"rel {st['rel']:.3e} absdeg {st['abs_degenerate']:.2e}", flush=True)

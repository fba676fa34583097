// tnrd_train.cuh -- stage backward of the TNRD diffusion on the GPU (SURVEY
// §8(f) rank 4: training.py:69-123 `_stage_backward`, imageops.py:75-127
// `conv2d_adjoint` / `patch_correlation`).
//
// For one stage t with u = u_prev, f, lambda and the upstream adjoint
// g_next = dL/du_next (reference names):
//
//   u~      = u - force(u)                      (prox)   training.py:79-83
//           = u - force(u) - lam (1/u - f^2/u^3) (projected)
//   g_t     = y * g_next, y = prox'(u~) or smooth_max'(u~)
//   grad_beta = lam * sum(dprox/dlam(u~) g_next)        (prox)
//             = -lam * sum((1/u - f^2/u^3) g_t)        (projected)
//   for each filter i:
//     z_i   = conv2d(u, k_i), phi_i = phi_i(z_i), phi'_i(z_i)
//     v_i   = conv2d_adjoint(g_t, rot180(k_i))
//     w1_i  = phi'_i * v_i
//     grad_weights[i][j] = -sum_P G_j(z_i[P]) v_i[P]
//     gk_i  = -rot180(patch_corr(u, w1_i)) - patch_corr(phi_i, g_t)
//             (the host maps gk_i to coefficient space: basis^T gk_i)
//     g_prev -= conv2d_adjoint(w1_i, k_i)          (filters ascending)
//   g_prev starts at g_t; the projected variant finally subtracts
//   lam (-1/u^2 + 3 f^2/u^4) g_t.
//
// Layout: whole-image maps per filter chunk in a stream-ordered workspace
// (training images are small: a 512^2 image x 48 filters x 5 maps = 252 MB).
// Kernels are direct (gather) formulations over the image -- the mirror
// padding's adjoint is folded in exactly, per output pixel, instead of the
// reference's full convolution + border fold -- and every reduction is
// two-pass in a fixed order (per-block partials in float64, then summed in
// block order), so results are bit-reproducible.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tnrd_stage.cuh"

namespace tnrd {
namespace train {

// half-sample mirror (one fold)
__device__ __forceinline__ int mir1(int j, int n) {
    return j < 0 ? -1 - j : (j >= n ? 2 * n - 1 - j : j);
}

// phi'(z) from the per-filter polynomial table (derivative of rbf_poly's
// interpolant: p'(x) / h)
__device__ __forceinline__ float rbf_poly_deriv(float z, const float* __restrict__ tabf,
                                                const StageArgs& p) {
    float t = fmaf(z, p.inv_h, p.t_off);
    t = fminf(fmaxf(t, 0.0f), p.tmax);
    const float r = t + 12582912.0f;
    const int j = __float_as_int(r) - 0x4B400000;
    const float x = t - (r - 12582912.0f);
    const float* c = tabf + rbf_lo_offset(j);
    const float4 lo = *reinterpret_cast<const float4*>(c);
    const float4 hi = *reinterpret_cast<const float4*>(c + 32);
    float acc = fmaf(7.0f * hi.w, x, 6.0f * hi.z);
    acc = fmaf(acc, x, 5.0f * hi.y);
    acc = fmaf(acc, x, 4.0f * hi.x);
    acc = fmaf(acc, x, 3.0f * lo.w);
    acc = fmaf(acc, x, 2.0f * lo.z);
    acc = fmaf(acc, x, lo.y);
    return acc * p.inv_h;
}

// phi'(z) as the reference writes it (influence.py:48-54 / training.py:90-94):
// sum_j w_j G_j(z) (mu_j - z) / gamma^2
__device__ __forceinline__ float rbf_direct_deriv(float z, const float* __restrict__ w,
                                                  const StageArgs& p) {
    const float inv_g2 = -2.0f * p.cE / 1.4426950408889634f;
    float s = 0.0f;
    for (int j = 0; j < p.M; ++j) {
        const float mu = fmaf((float)j, p.delta, p.mu0);
        const float d = z - mu;
        s = fmaf(w[j] * ex2f(d * d * p.cE), -d, s);
    }
    return s * inv_g2;
}

struct BwdArgs {
    StageArgs s;          // model tables of the stage (taps, tab, RBF constants, lam, variant)
    int H, W;             // dense images (ld = W)
    int m, kp;            // filter side, floats per filter in taps
    int f0, nf;           // filter chunk [f0, f0 + nf)
    const float* u;       // u_prev
    const float* f;       // observation
    const float* force;   // force(u_prev)
    const float* g_next;  // dL/du_next (NULL = zero)
    float* g_t;           // [H*W]
    float* z;             // [nf][H*W]
    float* phi;
    float* dphi;
    float* v;
    float* w1;
    float* adj;           // [nf][H*W] conv2d_adjoint(w1_i, k_i)
    float* g_prev;        // [H*W] in/out across chunks
    double* part;         // reduction partials
    int nblk;             // pixel blocks of the reductions
    int projected;
    int last_chunk;
};

constexpr int kRedPx = 256;  // pixels per reduction block (patch_corr_kernel)
constexpr int kSeg = 256;    // row-segment width of bwd_reduce_kernel blocks

// Pixel sets of the image-space kernels.  The interior rectangle (every
// m x m tap window inside the image: no mirror, no fold) runs branch-free;
// the border band (width r) runs the general mirror / preimage path.  Two
// launches keep every warp on one path.
struct PixelSet {
    int rt, rb, cl, cr;  // band widths: top, bottom, left, right
    int iw, ih;          // interior rectangle size
    int n;               // pixels in the set
    bool interior;
};

__host__ __device__ inline PixelSet pixel_set(int H, int W, int r, bool interior) {
    PixelSet ps;
    ps.rt = min(r, H);
    ps.rb = min(r, H - ps.rt);
    ps.cl = min(r, W);
    ps.cr = min(r, W - ps.cl);
    ps.ih = H - ps.rt - ps.rb;
    ps.iw = W - ps.cl - ps.cr;
    ps.interior = interior;
    ps.n = interior ? ps.ih * ps.iw : H * W - ps.ih * ps.iw;
    return ps;
}

// idx-th pixel of the set -> (Y, X)
__device__ __forceinline__ void set_pixel(const PixelSet& ps, int W, int idx, int& Y, int& X) {
    if (ps.interior) {
        Y = ps.rt + idx / ps.iw;
        X = ps.cl + idx % ps.iw;
        return;
    }
    const int top = ps.rt * W;
    if (idx < top) { Y = idx / W; X = idx % W; return; }
    idx -= top;
    const int side = ps.cl + ps.cr;
    const int mid = ps.ih * side;
    if (idx < mid) {
        Y = ps.rt + idx / side;
        const int c = idx % side;
        X = c < ps.cl ? c : W - ps.cr + (c - ps.cl);
        return;
    }
    idx -= mid;
    Y = ps.rt + ps.ih + idx / W;
    X = idx % W;
}

// g_t and the beta partials (per 256-pixel block, float64)
__global__ void __launch_bounds__(256) bwd_pointwise_kernel(const BwdArgs a) {
    __shared__ double red[256];
    const int n = a.H * a.W;
    const int i = blockIdx.x * 256 + threadIdx.x;
    double contrib = 0.0;
    if (i < n) {
        const float u = a.u[i], fv = a.f[i];
        const float gn = a.g_next ? a.g_next[i] : 0.0f;
        const float lam = a.s.lam;
        float gt;
        // the pointwise derivatives are evaluated in float64: the reference
        // formulas cancel (dprox/dlam subtracts two terms of similar size;
        // 1/u - f^2/u^3 vanishes at f = u), and the beta gradient sums them
        // over the image with further cancellation
        const double ud = u, fd = fv, ld = lam;
        if (a.projected) {
            const double rr = 1.0 / ud - (fd * fd) / (ud * ud * ud);
            const float ut = u - a.force[i] - (float)(ld * rr);
            const float tt = (ut - a.s.pfloor) * a.s.inv_tau;
            // stable logistic (diffusion.py:159-168)
            const float y = tt >= 0.0f ? 1.0f / (1.0f + expf(-tt)) : expf(tt) / (1.0f + expf(tt));
            gt = y * gn;
            contrib = -ld * rr * (double)gt;
        } else {
            const double ff = fmax(fd, (double)kFFloor);
            const double ut = (double)(u - a.force[i]);
            const double aa = 1.0 + 2.0 * ld;
            const double root = sqrt(ut * ut + 8.0 * aa * ld * ff * ff);
            const double y = (1.0 + ut / root) / (2.0 * aa);           // speckle.py:123-128
            const double x = (2.0 * ff * ff + 8.0 * ld * ff * ff) / (aa * root) -
                             (ut + root) / (aa * aa);                  // speckle.py:131-137
            gt = (float)(y * (double)gn);
            contrib = ld * x * (double)gn;
        }
        a.g_t[i] = gt;
    }
    red[threadIdx.x] = contrib;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) a.part[blockIdx.x] = red[0];
}

// z, phi, phi' of the chunk's filters (true convolution, mirror padded)
template <int MS, bool FAST>
__global__ void __launch_bounds__(256) bwd_maps_kernel(const BwdArgs a, const PixelSet ps) {
    const int n = a.H * a.W;
    const int idx = blockIdx.x * 256 + threadIdx.x;
    const int fi = blockIdx.y;
    if (idx >= ps.n) return;
    int Y, X;
    set_pixel(ps, a.W, idx, Y, X);
    const int i = Y * a.W + X;
    constexpr int r = MS / 2;
    const int gf = a.f0 + fi;
    const float* k = a.s.taps + (size_t)gf * a.kp;
    float z = 0.0f;
    if (ps.interior) {
#pragma unroll
        for (int p = -r; p <= r; ++p) {
            const float* row = a.u + (size_t)(Y - p) * a.W + X;
#pragma unroll
            for (int q = -r; q <= r; ++q) z = fmaf(k[(r + p) * MS + r + q], __ldg(row - q), z);
        }
    } else {
        for (int p = -r; p <= r; ++p) {
            const float* row = a.u + (size_t)mir1(Y - p, a.H) * a.W;
            for (int q = -r; q <= r; ++q) z = fmaf(k[(r + p) * MS + r + q], __ldg(row + mir1(X - q, a.W)), z);
        }
    }
    const float* tab = a.s.tab + (size_t)gf * a.s.tab_stride;
    const size_t o = (size_t)fi * n + i;
    a.z[o] = z;
    a.phi[o] = FAST ? rbf_poly(z, tab, a.s) : rbf_direct(z, tab, a.s);
    a.dphi[o] = FAST ? rbf_poly_deriv(z, tab, a.s) : rbf_direct_deriv(z, tab, a.s);
}

// (conv2d(., K)^T img)[Y, X] = sum_{p,q} K[r+p][r+q] sum over the preimages
// y of Y under y -> mir(y - p) (and likewise for x) of img[y][x]
__device__ __forceinline__ int preimages(int Y, int p, int n, int* out) {
    int c = 0;
    const int y0 = Y + p;                  // direct
    if (y0 >= 0 && y0 < n) out[c++] = y0;
    const int y1 = p - 1 - Y;              // mirrored below 0: y - p = -1 - Y
    if (y1 >= 0 && y1 < n) out[c++] = y1;
    const int y2 = 2 * n - 1 - Y + p;      // mirrored above n: y - p = 2n - 1 - Y
    if (y2 >= 0 && y2 < n) out[c++] = y2;
    return c;
}

// K[r+p][r+q] = kflip ? k[r-p][r-q] : k[r+p][r+q]
__device__ __forceinline__ float adjoint_at(const float* __restrict__ img, int H, int W, int Y, int X,
                                            const float* k, int m, bool kflip) {
    const int r = m / 2;
    float s = 0.0f;
    if (Y >= r && Y < H - r && X >= r && X < W - r) {
        // interior: every tap has exactly its direct preimage (Y + p, X + q)
        const float* base = img + (size_t)(Y - r) * W + (X - r);
        for (int a = 0; a < m; ++a) {
            const float* row = base + (size_t)a * W;
            const float* krow = kflip ? k + (m - 1 - a) * m : k + a * m;
            for (int b = 0; b < m; ++b) s = fmaf(kflip ? krow[m - 1 - b] : krow[b], __ldg(row + b), s);
        }
        return s;
    }
    for (int p = -r; p <= r; ++p) {
        int ys[3];
        const int ny = preimages(Y, p, H, ys);
        for (int q = -r; q <= r; ++q) {
            int xs[3];
            const int nx = preimages(X, q, W, xs);
            const float kk = kflip ? k[(r - p) * m + (r - q)] : k[(r + p) * m + (r + q)];
            float t = 0.0f;
            for (int a = 0; a < ny; ++a)
                for (int b = 0; b < nx; ++b) t += __ldg(img + (size_t)ys[a] * W + xs[b]);
            s = fmaf(kk, t, s);
        }
    }
    return s;
}

// interior adjoint with a compile-time filter side (fully unrolled taps)
template <int MS, bool KFLIP>
__device__ __forceinline__ float adjoint_interior(const float* __restrict__ img, int W, int Y, int X,
                                                  const float* __restrict__ k) {
    constexpr int r = MS / 2;
    const float* base = img + (size_t)(Y - r) * W + (X - r);
    float s = 0.0f;
#pragma unroll
    for (int a = 0; a < MS; ++a)
#pragma unroll
        for (int b = 0; b < MS; ++b)
            s = fmaf(KFLIP ? k[(MS - 1 - a) * MS + (MS - 1 - b)] : k[a * MS + b],
                     __ldg(base + (size_t)a * W + b), s);
    return s;
}

// v_i = conv2d_adjoint(g_t, rot180(k_i)), w1_i = phi'_i v_i
template <int MS>
__global__ void __launch_bounds__(256) bwd_v_kernel(const BwdArgs a, const PixelSet ps) {
    const int n = a.H * a.W;
    const int idx = blockIdx.x * 256 + threadIdx.x;
    const int fi = blockIdx.y;
    if (idx >= ps.n) return;
    int Y, X;
    set_pixel(ps, a.W, idx, Y, X);
    const int i = Y * a.W + X;
    const float* k = a.s.taps + (size_t)(a.f0 + fi) * a.kp;
    const float v = ps.interior ? adjoint_interior<MS, true>(a.g_t, a.W, Y, X, k)
                                : adjoint_at(a.g_t, a.H, a.W, Y, X, k, MS, true);
    const size_t o = (size_t)fi * n + i;
    a.v[o] = v;
    a.w1[o] = a.dphi[o] * v;
}

// A_i = conv2d_adjoint(w1_i, k_i) for every (pixel, filter) of the chunk
template <int MS>
__global__ void __launch_bounds__(256) bwd_adj_kernel(const BwdArgs a, const PixelSet ps) {
    const int n = a.H * a.W;
    const int idx = blockIdx.x * 256 + threadIdx.x;
    const int fi = blockIdx.y;
    if (idx >= ps.n) return;
    int Y, X;
    set_pixel(ps, a.W, idx, Y, X);
    const float* k = a.s.taps + (size_t)(a.f0 + fi) * a.kp;
    const float* w1 = a.w1 + (size_t)fi * n;
    a.adj[(size_t)fi * n + Y * a.W + X] = ps.interior ? adjoint_interior<MS, false>(w1, a.W, Y, X, k)
                                                      : adjoint_at(w1, a.H, a.W, Y, X, k, MS, false);
}

// g_prev = ((g_t - A_0) - A_1) - ... in filter order (training.py:111-113);
// the first chunk starts from g_t, the last adds the projected reaction term
__global__ void __launch_bounds__(256) bwd_gprev_kernel(const BwdArgs a) {
    const int n = a.H * a.W;
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    float g = a.f0 == 0 ? a.g_t[i] : a.g_prev[i];
    for (int fi = 0; fi < a.nf; ++fi) g -= a.adj[(size_t)fi * n + i];
    if (a.last_chunk && a.projected) {
        const float u = a.u[i], fv = a.f[i];
        g -= a.s.lam * (-1.0f / (u * u) + 3.0f * fv * fv / (u * u * u * u)) * a.g_t[i];
    }
    a.g_prev[i] = g;
}

// Parameter-gradient partials of one (row y, 256-column segment, filter)
// block, one output per warp (lanes over the segment, fixed xor-shuffle tree:
// deterministic).  With pad = mirror padding by r (np.pad symmetric):
//   o <  m^2       : C1[a][b] = sum_x pad(u)[y + a][x + b] w1[y][x]
//   o <  2 m^2     : C2[a][b] = sum_x pad(phi)[y + a][x + b] g_t[y][x]
//   o <  2 m^2 + M : GW[j]    = sum_x G_j(z[y][x]) v[y][x]
// (patch_correlation, imageops.py:109-127; the RBF design contraction,
// training.py:107).  The 2r+1 padded rows of u and phi, and the segment's
// w1, g_t, z, v, are staged in shared memory.
__device__ __forceinline__ float warp_sum(float s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// staged rows of bwd_reduce_kernel: logical column c at c + c / 8, so the
// 8-column windows of the 32 lanes start 9 floats apart (distinct banks)
__host__ __device__ constexpr int red_row_stride(int m) { return kSeg + 2 * (m / 2) + (kSeg + 2 * (m / 2)) / 8 + 1; }
__device__ __forceinline__ int pad8(int c) { return c + (c >> 3); }

// Parameter partials of one (image row, 256-column segment, filter): the
// m^2 kernel-gradient terms sum_x u[a][x + b] w1[x] and sum_x phi[a][x + b]
// g_t[x] as one work item per (term, tap row a) -- each lane owns 8
// consecutive columns, loads the row window once and keeps the m sums of
// that row in registers, then one xor tree per output -- and the M
// RBF-design terms sum_x G_j(z[x]) v[x], one item per output; items are
// dealt round-robin to the warps.  Fixed order throughout: bit-reproducible.
template <int MS>
__global__ void __launch_bounds__(256) bwd_reduce_kernel(const BwdArgs a, int nseg) {
    extern __shared__ float sm[];
    constexpr int R = MS / 2, MM = MS * MS;
    constexpr int SW = kSeg + 2 * R;           // staged row width
    constexpr int SWP = red_row_stride(MS);    // padded row stride
    static_assert(kSeg == 32 * 8, "one 8-column window per lane");
    const int n = a.H * a.W;
    const int fi = blockIdx.y;
    const int y = blockIdx.x / nseg, seg = blockIdx.x % nseg;
    const int x0 = seg * kSeg, nx = min(kSeg, a.W - x0);
    const int nout = 2 * MM + a.s.M;
    float* su = sm;                            // [MS][SWP]
    float* sp = su + MS * SWP;                 // [MS][SWP]
    float* sw1 = sp + MS * SWP;                // [kSeg] each
    float* sgt = sw1 + kSeg;
    float* sz = sgt + kSeg;
    float* sv = sz + kSeg;
    const size_t fo = (size_t)fi * n;
    for (int t = threadIdx.x; t < MS * SW; t += blockDim.x) {
        const int aa = t / SW, c = t % SW;
        const int xx = x0 + c - R;
        float uv = 0.0f, pv = 0.0f;
        if (c < nx + 2 * R) {
            const size_t off = (size_t)mir1(y + aa - R, a.H) * a.W + mir1(xx, a.W);
            uv = __ldg(a.u + off);
            pv = __ldg(a.phi + fo + off);
        }
        su[aa * SWP + pad8(c)] = uv;
        sp[aa * SWP + pad8(c)] = pv;
    }
    for (int t = threadIdx.x; t < kSeg; t += blockDim.x) {
        const bool ok = t < nx;
        const size_t off = (size_t)y * a.W + x0 + t;
        sw1[t] = ok ? __ldg(a.w1 + fo + off) : 0.0f;
        sgt[t] = ok ? __ldg(a.g_t + off) : 0.0f;
        sz[t] = ok ? __ldg(a.z + fo + off) : 0.0f;
        sv[t] = ok ? __ldg(a.v + fo + off) : 0.0f;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* part = a.part + ((size_t)fi * a.nblk + blockIdx.x) * nout;
    // work items: (term, tap row) pairs -- 8-column windows, MS sums each --
    // then the M RBF-design outputs, dealt round-robin to the warps
    const int nitems = 2 * MS + a.s.M;
    for (int it = warp; it < nitems; it += nw) {
        if (it < 2 * MS) {
            const int term = it / MS, aa = it - term * MS;
            const float* row = (term == 0 ? su : sp) + aa * SWP;
            const float* adj = term == 0 ? sw1 : sgt;   // zero beyond nx
            float w[8], v[8 + 2 * R], acc[MS];
#pragma unroll
            for (int k = 0; k < 8; ++k) w[k] = adj[8 * lane + k];
#pragma unroll
            for (int j = 0; j < 8 + 2 * R; ++j) v[j] = row[pad8(8 * lane + j)];
#pragma unroll
            for (int b = 0; b < MS; ++b) {
                acc[b] = 0.0f;
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[b] = fmaf(v[k + b], w[k], acc[b]);
            }
#pragma unroll
            for (int b = 0; b < MS; ++b) {
                const float s = warp_sum(acc[b]);
                if (lane == 0) part[term * MM + aa * MS + b] = s;
            }
        } else {
            const int o = 2 * MM + (it - 2 * MS);
            const float mu = fmaf((float)(o - 2 * MM), a.s.delta, a.s.mu0);
            float s = 0.0f;
            for (int x = lane; x < nx; x += 32) {
                const float d = sz[x] - mu;
                s = fmaf(ex2f(d * d * a.s.cE), sv[x], s);
            }
            s = warp_sum(s);
            if (lane == 0) part[o] = s;
        }
    }
}

// out[i][o] = sum over blocks b of part[i][b][o], one warp per output: lane
// l sums blocks l, l + 32, ... in order, then a fixed xor tree (float64)
__device__ __forceinline__ double warp_sum_d(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

__global__ void bwd_final_kernel(const double* __restrict__ part, double* out, int nf, int nblk, int nout) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= nf * nout) return;
    const int fi = t / nout, o = t - fi * nout;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += part[((size_t)fi * nblk + b) * nout + o];
    s = warp_sum_d(s);
    if (lane == 0) out[t] = s;
}

// drop-in conv2d_adjoint (imageops.py:90-106) for one kernel
__global__ void __launch_bounds__(256) conv2d_adjoint_kernel(const float* __restrict__ img, float* out,
                                                            int H, int W, const float* k, int m) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= H * W) return;
    const int Y = i / W, X = i - Y * W;
    out[i] = adjoint_at(img, H, W, Y, X, k, m, false);
}

// drop-in patch_correlation (imageops.py:109-127): per 256-pixel block
// partials of C[a][b] = sum_P base[mir(P + (a - r, b - r))] adj[P]
__global__ void __launch_bounds__(128) patch_corr_kernel(const float* __restrict__ base,
                                                        const float* __restrict__ adj, int H, int W,
                                                        int m, double* part) {
    const int n = H * W, mm = m * m, r = m / 2;
    const int blk = blockIdx.x;
    const int P0 = blk * kRedPx, P1 = min(n, P0 + kRedPx);
    for (int o = threadIdx.x; o < mm; o += blockDim.x) {
        const int da = o / m - r, db = o % m - r;
        float s = 0.0f;
        for (int P = P0; P < P1; ++P) {
            const int Y = P / W, X = P - Y * W;
            s = fmaf(__ldg(base + (size_t)mir1(Y + da, H) * W + mir1(X + db, W)), __ldg(adj + P), s);
        }
        part[(size_t)blk * mm + o] = s;
    }
}

}  // namespace train
}  // namespace tnrd

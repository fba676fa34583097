// tnrd_stage.cuh -- fused TNRD diffusion stage for sm_100a.
//
// One launch = one stage of diffusion_step (reference diffusion.py:184-194)
// over a batch of images:
//
//   z_i   = conv2d(u, k_i)                 imageops.py:53-72 (mirror padded)
//   phi_i = sum_j w_ij exp(-(z_i-mu_j)^2/(2 gamma^2))   influence.py:40-45
//   force = sum_i conv2d(phi_i, rot180(k_i))   diffusion.py:178-180 (phi is
//           mirror padded itself, NOT the exact adjoint)
//   u'    = prox_idiv(u - force, f, lam)   speckle.py:111-121
//
// B200 mapping (see DESIGN.md for the derivation):
//   * a CTA owns a TH x TW output tile; u is staged in shared memory with a
//     2r halo, phi for F filters at a time with an r halo;
//   * filters are processed in groups of F; the group's taps and RBF tables
//     are prefetched into shared memory with cp.async one group ahead;
//   * forward pass: each work item = one filter x RF x 4 phi block; the 49
//     taps live in registers, u rows are read as float4;
//   * the RBF phi_i is evaluated from a per-filter piecewise degree-7
//     polynomial table (float64 Chebyshev fit on the host, error ~1e-9 of
//     sum|w|): 2 conflict-free LDS.128 + 7 FFMA per response instead of
//     M=63 exponentials;
//   * the large-tile default kernels (stage_kernel_pt / _split_pt, DESIGN.md
//     4.9-4.10) instead read the taps from the kernel parameter space
//     (uniform datapath) and phi from a cubic table (one LDS.128 + 3 FFMA)
//     fetched per filter group with cp.async.bulk on an mbarrier;
//   * phi halos that fall outside the image are filled by mirroring the
//     in-image phi values (reference pads phi itself, diffusion.py:180);
//   * backward pass: each thread owns an RB x 4 output block for half of
//     the group's filters and keeps its partial force in registers across
//     all groups; the two halves are summed once in the epilogue;
//   * epilogue: u~ = u - force, cancellation-free prox, non-finite flag,
//     f validation (stage 0), store;
//   * small grids (one 512^2 image) run the split kernel instead: units of
//     (tile, filter group) over a persistent grid, partial forces reduced in
//     a fixed order by the tile's last unit (stage_kernel_split).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tnrd {

constexpr int kF = 4;          // filters per group
constexpr int kPolyDeg = 7;    // RBF interpolant degree per interval
constexpr int kPolyN = kPolyDeg + 1;  // coefficients per interval
constexpr int kPolySub = 2;    // intervals per min(delta, gamma)
// cubic table (parameter-space-taps kernels, rbf_cubic_s): 10 intervals per
// min(delta, gamma): interpolation error ~1e-7 of sum|w| (fp32 resolution
// of phi); at most kMaxCubicStride floats per filter (a single-buffered
// 2-filter group table then fits beside 2 CTAs per SM)
constexpr double kCubicSub = 10.0;
constexpr int kMaxCubicStride = 4096;
constexpr float kFFloor = 1e-6f;  // speckle.py:21

__host__ __device__ constexpr int round_up(int x, int a) { return (x + a - 1) / a * a; }

// u-tile row stride: at least `need`, a multiple of 4 floats, and chosen so
// that a step of `rows` rows shifts the bank by 4*nbx (mod 32 banks): the
// float4 loads of consecutive forward blocks that straddle a block-row
// boundary then hit disjoint banks.
__host__ __device__ constexpr int padded_stride(int need, int rows, int nbx) {
    int s = round_up(need, 4);
    for (int k = 0; k < 8; ++k, s += 4)
        if ((rows * s - 4 * nbx) % 32 == 0) return s;
    return round_up(need, 4);
}

struct StageArgs {
    const float* u_in;
    const float* f;
    float* u_out;
    const float* taps;   // [nk_pad][KP]  reference k_i (row-major a,b)
    const float* tab;    // [nk_pad][tab_stride] RBF table (fast: Horner A, generic: w)
    int64_t ld;          // elements between rows
    int64_t img_stride;  // elements between images
    int H, W;
    int ngroups;         // filter groups (of kF, or tc::kG on the tensor-core path)
    int nk;              // real filters (padding filters are zero)
    int tab_stride;      // floats per filter in tab
    // prox (speckle.py:111-121): a = 1 + 2 lam
    float lam4;          // 4 lam
    float c8;            // 8 a lam
    float inv2a;         // 1 / (2a)
    // RBF: polynomial table (default) -- t = z / h + t_off, clamp [0, tmax];
    // interval j at tab[8 j], halves swapped when bit 2 of j is set
    float inv_h;
    uint32_t tab_bias;   // -(0x4B400000 << 5) mod 2^32, a runtime value so ptxas keeps it in the table base register
    int tab_ni;
    float t_off;
    float tmax;
    // RBF: cubic table (parameter-space-taps kernels): interval j at tab3[4 j]
    const float* tab3;   // [nk_pad][tab3_stride]
    int tab3_stride;     // floats per filter (0: no cubic table)
    uint32_t tab3_bias;  // -(0x4B400000 << 4) mod 2^32
    float inv_h3;
    float t_off3;
    float tmax3;
    // RBF: direct all-centre sum (fallback for very large tables)
    float delta;
    float cE;            // -log2(e) / (2 gamma^2)
    float mu0;
    int M;
    // projected comparison variant (diffusion.py:149-168, 197-224)
    float lam;           // lambda of the stage
    float pfloor;        // projection floor
    float tau;           // PROJECTION_KNEE * floor
    float inv_tau;
    float u0_floor;      // initial_state floor: 1e-6 (prox) or the projection floor
    uint32_t flags;
    int stage;
    uint32_t* status;    // [0] first non-finite stage (atomicMin), [1] f flags (atomicAnd ~bit)
    float* force_out;    // optional second output: the force (tnrd_stage_force), same layout as u_out
    // stage_kernel_cl*: CTAs per cluster (= gridDim.x), groups per rank and
    // ranks with one more, tiles per image row (blockIdx.y = tile_y * cl_tiles_x + tile_x)
    int cluster, cl_gper, cl_gextra, cl_tiles_x;
};

// Debug bounds mode (-DTNRD_BOUNDS, tools/bounds_run.sh): every shared-memory
// index computed at run time -- forward / backward block extents, RBF table
// lookups, the phi fix-up, split / cluster partial stores -- and the image
// coordinates of the global accesses are checked against their buffer;
// violations are counted (first one kept) in g_bounds_fail and read back with
// tnrd_bounds_failures().  compute-sanitizer is closed on the GPU pool, so
// this build is the memory-safety evidence: the GPU test suite must finish
// with zero violations (profiles/r02_bounds).
#ifdef TNRD_BOUNDS
__device__ unsigned int g_bounds_fail[4];   // count, kind, value, limit of the first
__device__ __forceinline__ void bounds_fail(unsigned kind, unsigned v, unsigned lim) {
    if (atomicAdd(&g_bounds_fail[0], 1u) == 0u) {
        g_bounds_fail[1] = kind; g_bounds_fail[2] = v; g_bounds_fail[3] = lim;
    }
}
#define TNRD_ASSERT(cond, kind, v, lim) do { if (!(cond)) bounds_fail(kind, (unsigned)(v), (unsigned)(lim)); } while (0)
#else
#define TNRD_ASSERT(cond, kind, v, lim) do { } while (0)
#endif

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 128-bit shared load that the compiler may not narrow (a narrowed LDS.64
// tail breaks the 8-lane conflict-free phase pattern of the row loads).
// The "memory" clobber keeps it ordered with the CTA barriers and the
// shared stores of other phases (without it the load may be hoisted across
// __syncthreads and read a previous filter group's phi).
__device__ __forceinline__ float4 lds128(const float* ptr) {
    float4 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(ptr));
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a)
                 : "memory");
    return v;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// I-divergence prox (speckle.py:111-121): u' = (u~ + sqrt(u~^2 + 8 a lam
// f^2)) / (2a), f floored at 1e-6, evaluated cancellation-free for u~ < 0
// as 4 lam f^2 / (root - u~).  The reference squares in float64, so it
// stays finite wherever its result fits; fp32 squares overflow once |u~| or
// f exceeds ~1e19.  When |u~| > 2^60 or 8 a lam f^2 overflows (rare: the
// branch is uniform in practice) u~ and f are scaled by an exact power of
// two 2^-E, E = exponent of max(|u~|, f), and the result is scaled back:
// finite whenever the true result fits in fp32; non-finite for a non-finite
// u~ (the reference's inf / nan) or a result beyond the fp32 range.
__device__ __forceinline__ float prox_idiv_f(float ut, float fv, float lam4, float c8, float inv2a) {
    const float ff = fmaxf(fv, kFFloor);
    const float fl2 = ff * ff;
    const float q = c8 * fl2;
    if (fabsf(ut) <= 1.152921504606847e18f && q <= 3.4028234663852886e38f) {   // 2^60, FLT_MAX
        const float root = sqrtf(fmaf(ut, ut, q));
        return ut >= 0.0f ? (ut + root) * inv2a : (lam4 * fl2) / (root - ut);
    }
    if (!(fabsf(ut) < __int_as_float(0x7f800000))) return ut - ut;   // +-inf, nan -> nan
    // s = 2^-E (exponent field 254 - e, at least 1), 1/s = 2^E exactly
    const int eb = __float_as_int(fmaxf(fabsf(ut), ff)) & 0x7f800000;
    const int sb = max(0x7f000000 - eb, 0x00800000);
    const float s = __int_as_float(sb);
    const float inv_s = __int_as_float(0x7f000000 - sb);
    const float uts = ut * s, ffs = ff * s;
    const float fs2 = ffs * ffs;
    const float root = sqrtf(fmaf(uts, uts, c8 * fs2));
    // u~ < 0: 4 lam f^2 / (root - u~) = 4 lam f * (f s / ((root - u~) s)):
    // no square of the (possibly underflowing) scaled f
    return ut >= 0.0f ? ((uts + root) * inv2a) * inv_s : (lam4 * ff) * (ffs / (root - uts));
}

// Reaction step of one pixel: the I-divergence prox above or, with
// TNRD_STAGE_PROJECTED, the projected comparison variant
// u' = smooth_max(u - force - lam (1/u - f^2/u^3), floor) with
// smooth_max(x, c) = c + tau log(1 + exp((x - c)/tau)), tau = 0.01 c
// (diffusion.py:149-168, 197-216); f^2/u^3 is formed as (f/u)^2 / u so it
// does not overflow before the float64 reference would.  `fv` is the raw
// observation.
__device__ __forceinline__ float reaction(float u, float force, float fv, const StageArgs& p) {
    if (p.flags & 0x20u) {
        const float iu = 1.0f / u;
        const float fu = fv * iu;
        const float ut = u - force - p.lam * (iu - fu * fu * iu);
        const float x = (ut - p.pfloor) * p.inv_tau;
        return fmaf(p.tau, fmaxf(x, 0.0f) + log1pf(expf(-fabsf(x))), p.pfloor);
    }
    return prox_idiv_f(u - force, fv, p.lam4, p.c8, p.inv2a);
}

// Half-sample symmetric reflection (np.pad mode="symmetric", one fold) and
// clamp: positions further out than one fold only feed discarded outputs.
__device__ __forceinline__ int mirror_clamp(int j, int n) {
    j = j < 0 ? -1 - j : j;
    j = j >= n ? 2 * n - 1 - j : j;
    return min(max(j, 0), n - 1);
}

// phi(z) from the per-filter piecewise polynomial table (default path).
//   The host samples phi_i(z) = sum_j w_ij exp(-(z-mu_j)^2/(2 gamma^2)) in
//   float64 at 8 Chebyshev nodes of every interval of width
//   h = min(delta, gamma) / 2 covering [mu_0 - 7 gamma, mu_{M-1} + 7 gamma]
//   and stores the degree-7 interpolant's monomial coefficients in the local
//   variable x in [-1/2, 1/2].  Layout: blocks of 8 intervals, 64 floats
//   each -- c0..c3 of the 8 intervals, then c4..c7 -- so 8 lanes reading 8
//   consecutive intervals hit 8 distinct bank quads and the second half is
//   an immediate +128 B.  Interpolation error ~1e-9 * sum|w| (checked on the
//   host at model creation); no MUFU, 2 LDS.128 + 7 FFMA
//   per response instead of 63 exp + 63 FMA.
__host__ __device__ constexpr int rbf_lo_offset(int j) { return (j >> 3) * 64 + (j & 7) * 4; }

__device__ __forceinline__ float rbf_horner(float x, float4 lo, float4 hi) {
    float acc = fmaf(hi.w, x, hi.z);
    acc = fmaf(acc, x, hi.y);
    acc = fmaf(acc, x, hi.x);
    acc = fmaf(acc, x, lo.w);
    acc = fmaf(acc, x, lo.z);
    acc = fmaf(acc, x, lo.y);
    return fmaf(acc, x, lo.x);
}

// generic-pointer version (tables in global or shared memory)
__device__ __forceinline__ float rbf_poly(float z, const float* __restrict__ tabf,
                                          const StageArgs& p) {
    float t = fmaf(z, p.inv_h, p.t_off);
    t = fminf(fmaxf(t, 0.0f), p.tmax);
    const float r = t + 12582912.0f;                 // rint(t) in the low bits
    const int j = __float_as_int(r) - 0x4B400000;
    const float x = t - (r - 12582912.0f);           // in [-1/2, 1/2]
    const float* c = tabf + rbf_lo_offset(j);
    return rbf_horner(x, *reinterpret_cast<const float4*>(c), *reinterpret_cast<const float4*>(c + 32));
}

// shared-memory version for the stage kernels: `tb` = the table's shared
// address + p.tab_bias (= -(0x4B400000 << 5), a runtime value so ptxas keeps
// it folded in the register); with b = the rounded float's bits, interval
// j = b - 0x4B400000 starts at tb + (b >> 3) * 128 + b * 16 (3 integer
// instructions, both halves at immediate offsets)
__device__ __forceinline__ uint32_t rbf_table_base(const float* tabf, const StageArgs& p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(tabf)) + p.tab_bias;
}

__device__ __forceinline__ float rbf_poly_s(float z, uint32_t tb, const StageArgs& p) {
    float t = fmaf(z, p.inv_h, p.t_off);
    t = fminf(fmaxf(t, 0.0f), p.tmax);
    const float r = t + 12582912.0f;
    const float x = t - (r - 12582912.0f);
    const uint32_t b = static_cast<uint32_t>(__float_as_int(r));
    const uint32_t a = ((b >> 3) << 7) + (b << 4) + tb;
    TNRD_ASSERT((a - (tb - p.tab_bias)) + 144u <= 4u * (uint32_t)p.tab_stride && !(a & 15u), 3, a - (tb - p.tab_bias), 4 * p.tab_stride);
    float4 lo, hi;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%8];\n\t"
                 "ld.shared.v4.f32 {%4, %5, %6, %7}, [%8+128];"
                 : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
                 : "r"(a)
                 : "memory");
    return rbf_horner(x, lo, hi);
}

// cubic table (parameter-space-taps kernels): interval j = one float4
// c0..c3 at tb3 + 16 j bytes (`tb3` = the table's shared address +
// p.tab3_bias); 8 lanes with consecutive intervals hit 8 distinct bank
// quads.  One 128-bit load + 3 FFMA per response (the degree-7 table needs
// two loads + 7 FFMA; measured on B200 the second load's latency, not the
// FFMAs, is what the forward waits on).
__device__ __forceinline__ float rbf_cubic_s(float z, uint32_t tb3, const StageArgs& p) {
    float t = fmaf(z, p.inv_h3, p.t_off3);
    t = fminf(fmaxf(t, 0.0f), p.tmax3);
    const float r = t + 12582912.0f;
    const float x = t - (r - 12582912.0f);
    const uint32_t a = (static_cast<uint32_t>(__float_as_int(r)) << 4) + tb3;
    TNRD_ASSERT((a - (tb3 - p.tab3_bias)) + 16u <= 4u * (uint32_t)p.tab3_stride && !(a & 15u), 3, a - (tb3 - p.tab3_bias), 4 * p.tab3_stride);
    float4 c;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(c.x), "=f"(c.y), "=f"(c.z), "=f"(c.w)
                 : "r"(a)
                 : "memory");
    return fmaf(fmaf(fmaf(c.w, x, c.z), x, c.y), x, c.x);
}

// phi(z) as the reference writes it: all M centres (generic bandwidths).
__device__ __forceinline__ float rbf_direct(float z, const float* __restrict__ w,
                                            const StageArgs& p) {
    float s = 0.0f;
    for (int j = 0; j < p.M; ++j) {
        const float d = z - fmaf((float)j, p.delta, p.mu0);
        s = fmaf(w[j], ex2f(d * d * p.cE), s);
    }
    return s;
}

template <int MS, int TH, int TW, int RF, int RB, int NT, int F = kF>
struct StageCfg {
    static constexpr int R = MS / 2;
    static constexpr int PH = round_up(TH + 2 * R, RF);  // phi rows computed
    static constexpr int PW = round_up(TW + 2 * R, 4);   // phi cols computed (stride)
    static constexpr int UR = PH + 2 * R;                // u rows staged
    static constexpr int US = padded_stride(PW + round_up(2 * R, 4), RF, PW / 4);  // u row stride
    static constexpr int NV = (4 + 2 * R + 3) / 4;       // float4 per row segment
    static constexpr int KK = MS * MS;
    static constexpr int KP = round_up(KK, 4);
    static constexpr int NBX = PW / 4;                   // forward blocks per row
    static constexpr int NBY = PH / RF;
    static constexpr int NBLK = NBX * NBY;               // forward blocks per filter
    static constexpr int TPF = NT / F;                   // forward threads per filter
    static_assert(TPF * F == NT, "forward threads must split evenly over the filters");
    static constexpr int OBX = TW / 4;                   // output blocks
    static constexpr int OBY = TH / RB;
    static constexpr int NSPLIT = NT / (OBX * OBY);      // bwd filter split
    static_assert(OBX * OBY * NSPLIT == NT && F % NSPLIT == 0,
                  "output blocks x filter split must cover the CTA");
    static_assert(TW % 4 == 0 && TH % RB == 0, "tile shape");
    static constexpr int SU = UR * US;
    static constexpr int SPHI = PH * PW;
    // shared layout (floats): u | phi[F] | taps[2][F*KP] | tab[2][F*tab_stride]
    static size_t smem_bytes(int tab_stride) {
        return sizeof(float) * (size_t)(SU + F * SPHI + 2 * F * KP + 2 * F * tab_stride);
    }
};

// ---- building blocks shared by the tile kernel and the split kernel --------

// u tile with a 2r halo, mirrored at image edges (or read from the halo rows
// of a row strip), floored on the first stage (initial_state,
// diffusion.py:219-224)
// COHERENT: u was written earlier in the same kernel (the fused dataflow
// kernel) -- read through L2 (ld.global.cg), not the read-only path
template <class C, int NT, bool COHERENT = false>
__device__ __forceinline__ void stage_u_tile(const StageArgs& p, float* sU, const float* __restrict__ uin,
                                             int Y0, int X0, bool top_halo, bool bot_halo, int tid) {
    constexpr int R = C::R;
    // all of the tile's loads in flight at once (one L2 round trip, not three)
    constexpr int B = (C::SU + NT - 1) / NT < 32 ? (C::SU + NT - 1) / NT : 32;
    const bool floor_in = p.flags & 0x1u;
    for (int i0 = tid; i0 < C::SU; i0 += B * NT) {
        float v[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const int i = i0 + j * NT;
            if (i < C::SU) {
                const int uy = i / C::US, ux = i - uy * C::US;
                int Y = Y0 - 2 * R + uy;
                const int X = mirror_clamp(X0 - 2 * R + ux, p.W);
                if (Y < 0) Y = top_halo ? max(Y, -2 * R) : mirror_clamp(Y, p.H);
                else if (Y >= p.H) Y = bot_halo ? min(Y, p.H - 1 + 2 * R) : mirror_clamp(Y, p.H);
                TNRD_ASSERT(X >= 0 && X < p.W && Y >= (top_halo ? -2 * R : 0) && Y < p.H + (bot_halo ? 2 * R : 0), 5, Y, p.H);
                v[j] = COHERENT ? __ldcg(uin + (int64_t)Y * p.ld + X) : __ldg(uin + (int64_t)Y * p.ld + X);
            }
        }
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const int i = i0 + j * NT;
            if (i < C::SU) sU[i] = floor_in ? fmaxf(v[j], p.u0_floor) : v[j];
        }
    }
}

template <class C, int F, int NT>
__device__ __forceinline__ void prefetch_group(const StageArgs& p, float* sTap, float* sTab, int g,
                                               int buf, int tid) {
    const int tabsz = F * p.tab_stride;
    const float* gt = p.taps + (size_t)g * F * C::KP;
    float* st = sTap + buf * F * C::KP;
    for (int i = tid; i < F * C::KP / 4; i += NT) cp_async16(st + 4 * i, gt + 4 * i);
    const float* gb = p.tab + (size_t)g * tabsz;
    float* sb = sTab + buf * tabsz;
    for (int i = tid; i < tabsz / 4; i += NT) cp_async16(sb + 4 * i, gb + 4 * i);
    cp_async_commit();
}

template <class C>
__device__ __forceinline__ void load_taps(const float* tap, float (&k)[C::KK]) {
    const float4* t4 = reinterpret_cast<const float4*>(tap);
#pragma unroll
    for (int q = 0; q < C::KP / 4; ++q) {
        const float4 v = t4[q];
        if (4 * q + 0 < C::KK) k[4 * q + 0] = v.x;
        if (4 * q + 1 < C::KK) k[4 * q + 1] = v.y;
        if (4 * q + 2 < C::KK) k[4 * q + 2] = v.z;
        if (4 * q + 3 < C::KK) k[4 * q + 3] = v.w;
    }
}

// forward of one RF x 4 phi block of one filter: z = conv(u, k), phi = rbf(z).
// K is the filter's taps: a register array (taps staged in shared memory) or
// a pointer into the kernel's parameter space (TapBlock: warp-uniform, read
// by the uniform datapath -- LDCU + FFMA with a uniform-register operand --
// so the taps hold no per-thread registers).
// RBF lookups interleaved with the convolution (forward_block, forward_block_fp)
#ifndef TNRD_FWD_INTERLEAVE
#define TNRD_FWD_INTERLEAVE 1
#endif

// phi = rbf(z) of one 4-wide row (cubic table / degree-7 table / direct sum)
template <bool FAST, bool CUBIC>
__device__ __forceinline__ float4 rbf_row(const float (&z)[4], uint32_t tb, const float* tabf, const StageArgs& p) {
    float4 o;
    if (CUBIC) {
        o.x = rbf_cubic_s(z[0], tb, p); o.y = rbf_cubic_s(z[1], tb, p);
        o.z = rbf_cubic_s(z[2], tb, p); o.w = rbf_cubic_s(z[3], tb, p);
    } else if (FAST) {
        o.x = rbf_poly_s(z[0], tb, p); o.y = rbf_poly_s(z[1], tb, p);
        o.z = rbf_poly_s(z[2], tb, p); o.w = rbf_poly_s(z[3], tb, p);
    } else {
        o.x = rbf_direct(z[0], tabf, p); o.y = rbf_direct(z[1], tabf, p);
        o.z = rbf_direct(z[2], tabf, p); o.w = rbf_direct(z[3], tabf, p);
    }
    return o;
}

// forward of one RF x 4 phi block of one filter: z = conv(u, k), phi = rbf(z).
// K is the filter's taps: a register array (taps staged in shared memory) or
// a pointer into the kernel's parameter space (TapBlock: warp-uniform, read
// by the uniform datapath -- LDCU + FFMA with a uniform-register operand --
// so the taps hold no per-thread registers).  TNRD_FWD_INTERLEAVE: each
// output row's lookups right after its last input row, its store one input
// row later (see forward_block_fp); else the lookups after the convolution,
// stored in batches of BATCH_ROWS.
template <class C, int MS, int RF, bool FAST, int BATCH_ROWS, bool CUBIC = false, class K>
__device__ __forceinline__ void forward_block(const StageArgs& p, const float* sU, float* phif,
                                              const K& k, uint32_t tb, const float* tabf, int blk) {
    constexpr int R = C::R;
    const int by = blk / C::NBX;
    const int bx = blk - by * C::NBX;
    const int x0 = bx * 4, y0 = by * RF;
    TNRD_ASSERT(blk >= 0 && blk < C::NBLK && y0 + RF + 2 * R <= C::UR && x0 + 4 * C::NV <= C::US &&
                y0 + RF <= C::PH && x0 + 4 <= C::PW, 1, blk, C::NBLK);
    float* dst = phif + y0 * C::PW + x0;
    float acc[RF][4];
#pragma unroll
    for (int r = 0; r < RF; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0f;
    float4 prev;
#pragma unroll
    for (int rr = 0; rr < RF + 2 * R; ++rr) {
        float v[4 * C::NV];
        const float* src = sU + (y0 + rr) * C::US + x0;
#pragma unroll
        for (int q = 0; q < C::NV; ++q) {
            const float4 t = lds128(src + 4 * q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
#pragma unroll
        for (int a = 0; a < MS; ++a) {
            const int ro = rr - a;
            if (ro >= 0 && ro < RF) {
#pragma unroll
                for (int b = 0; b < MS; ++b) {
                    // true convolution == correlation with rot180(k)
                    const float kk = k[(MS - 1 - a) * MS + (MS - 1 - b)];
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[ro][c] = fmaf(kk, v[c + b], acc[ro][c]);
                }
            }
        }
        if constexpr (TNRD_FWD_INTERLEAVE) {
            const int r = rr - 2 * R;   // output row completed by this input row
            if (r >= 1) *reinterpret_cast<float4*>(dst + (r - 1) * C::PW) = prev;
            if (r >= 0) prev = rbf_row<FAST, CUBIC>(acc[r], tb, tabf, p);
        }
    }
    if constexpr (TNRD_FWD_INTERLEAVE) {
        *reinterpret_cast<float4*>(dst + (RF - 1) * C::PW) = prev;
    } else {
        // BATCH_ROWS = RF: all RF x 4 table lookups before the first phi
        // store (the lookups are ordered asm loads with a memory clobber, so
        // a store between rows caps the lookups in flight at one row's four)
        float4 o[RF];
#pragma unroll
        for (int r = 0; r < RF; ++r) {
            o[r] = rbf_row<FAST, CUBIC>(acc[r], tb, tabf, p);
            if ((r + 1) % BATCH_ROWS == 0 || r == RF - 1) {
#pragma unroll
                for (int q = r - (r % BATCH_ROWS); q <= r; ++q)
                    *reinterpret_cast<float4*>(dst + q * C::PW) = o[q];
            }
        }
    }
}

// forward: z = conv(u, k) on the phi region, phi = rbf(z); TPF threads per
// filter, each with the filter's taps in registers
template <class C, int MS, int RF, int F, bool FAST, int BATCH_ROWS = RF>
__device__ __forceinline__ void forward_group(const StageArgs& p, const float* sU, float* sPhi,
                                              const float* tapg, const float* tabg, int tid) {
    const int fi = tid / C::TPF;
    float k[C::KK];
    load_taps<C>(tapg + fi * C::KP, k);
    const float* tabf = tabg + fi * p.tab_stride;
    const uint32_t tb = rbf_table_base(tabf, p);
    float* phif = sPhi + fi * C::SPHI;
    for (int blk = tid - fi * C::TPF; blk < C::NBLK; blk += C::TPF)
        forward_block<C, MS, RF, FAST, BATCH_ROWS>(p, sU, phif, k, tb, tabf, blk);
}

// ---- FFMA2 (fma.rn.f32x2, sm_100): two IEEE fma.rn lanes per instruction --
// FFMA2 reaches the FFMA FLOP peak at half the issue slots (measured on
// B200, tools/probes/ffma2_probe.cu: 71.6 vs 72.3 TFLOP/s), which leaves the
// slots for the shared-memory loads and the RBF.  The parameter-space-taps
// kernels (m <= 7) pair two OUTPUT ROWS of a block: lanes (row 2q, row
// 2q + 1) share the input value (a broadcast register operand) and take two
// taps from a uniform register pair.  Each lane is the same fma.rn on the
// same operands in the same order as the scalar loop, so results are
// bit-identical to the FFMA kernels.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float f2_lo(f2_t v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    (void)hi;
    return lo;
}
__device__ __forceinline__ float f2_hi(f2_t v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    (void)lo;
    return hi;
}
// d = a * b + c per lane
__device__ __forceinline__ f2_t ffma2(f2_t a, f2_t b, f2_t c) {
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

// Pair-tap layout of one filter (parameter space, m <= 7): for tap rows
// A = 1..MS-1 and columns B, Q[A][B] = (k[A][B], k[A-1][B]) at float2 index
// (A-1) MS + B; single taps are halves of pairs (k[0][B] = Q[1][B].y).
template <int MS>
struct PairTaps {
    static constexpr bool kOn = MS >= 3 && MS <= 7;
    static constexpr int kFloats = round_up(2 * (MS - 1) * MS, 4);   // per filter
};
template <int MS>
__device__ __forceinline__ float2 qpair(const float* kq, int A, int B) {
    return reinterpret_cast<const float2*>(kq)[(A - 1) * MS + B];
}
template <int MS>
__device__ __forceinline__ float qsingle(const float* kq, int A, int B) {
    return A >= 1 ? qpair<MS>(kq, A, B).x : qpair<MS>(kq, 1, B).y;
}

// Tap layouts of the parameter-space kernels (TM = tap mode):
//   0: row-major k per filter (KP floats), scalar FFMA
//   1: row pairs per filter (PairTaps), FFMA2 over output-row pairs
//   2: per group of F = 2 filters, the forward's FILTER pairs
//      FP[a][b] = (kf_f0[a][b], kf_f1[a][b]) (kf = rot180 k, 2 MS^2 floats
//      rounded to 4), then each filter's row pairs for the backward.  The
//      forward computes both filters of the group per thread (one u-row load
//      feeds both), FFMA2 over the filter pair; the backward runs row pairs.
//   3: the filter pairs FP only (fits the parameter space for m = 9, Nk = 80);
//      the backward runs scalar FFMA on the halves of FP (k = rot180 kf).
template <int MS, int KP, int F, int TM>
struct TapLayout {
    static constexpr int KQ = PairTaps<MS>::kFloats;
    static constexpr int FPF = round_up(2 * MS * MS, 4);
    static constexpr int per_filter = TM == 0 ? KP : (TM == 3 ? 1 : KQ);   // backward taps per filter
    static constexpr int bwd0 = TM == 2 ? FPF : 0;                         // backward taps offset in a group
    static constexpr int group = TM == 2 ? FPF + F * KQ : (TM == 3 ? FPF : F * per_filter);
    static_assert(TM < 2 || F == 2, "filter-pair forward needs 2 filters per group");
    static_assert(TM == 0 || TM == 3 || PairTaps<MS>::kOn, "row pairs need 3 <= m <= 7");
};

// tap k_fi[i] (i = a MS + b) of a filter-pair block FP (TM 3): the rot180
// partner kf[MS^2 - 1 - i], lane fi; `fp` is already offset by fi
template <int MS>
struct FpTap {
    const float* fp;
    __device__ __forceinline__ float operator[](int i) const { return fp[2 * (MS * MS - 1 - i)]; }
};

// forward of both filters of a group (TM 2, 3): one RF x 4 block, z of
// filter 0 / 1 in the low / high lane of each FFMA2 (same fma.rn chain per
// filter as the scalar forward_block, so the same bits).  Output row r is
// complete after input row r + 2R: with TNRD_FWD_INTERLEAVE its RBF lookups
// are issued right there and its phi stored one input row later, so the
// lookup latency hides under the remaining rows' FFMA2s (instead of a
// lookup-only tail after the convolution).
template <class C, int MS, int RF, int BATCH_ROWS>
__device__ __forceinline__ void forward_block_fp(const StageArgs& p, const float* sU, float* phi0, float* phi1,
                                                 const float* kfp, uint32_t tb0, uint32_t tb1, int blk) {
    constexpr int R = C::R;
    const int by = blk / C::NBX;
    const int bx = blk - by * C::NBX;
    const int x0 = bx * 4, y0 = by * RF;
    TNRD_ASSERT(blk >= 0 && blk < C::NBLK && y0 + RF + 2 * R <= C::UR && x0 + 4 * C::NV <= C::US &&
                y0 + RF <= C::PH && x0 + 4 <= C::PW, 1, blk, C::NBLK);
    float* d0 = phi0 + y0 * C::PW + x0;
    float* d1 = phi1 + y0 * C::PW + x0;
    f2_t acc2[RF][4];
#pragma unroll
    for (int r = 0; r < RF; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc2[r][c] = 0ull;
    float4 p0, p1;   // interleave: phi of the previous completed row, stored one row later
#pragma unroll
    for (int rr = 0; rr < RF + 2 * R; ++rr) {
        float v[4 * C::NV];
        const float* src = sU + (y0 + rr) * C::US + x0;
#pragma unroll
        for (int q = 0; q < C::NV; ++q) {
            const float4 t = lds128(src + 4 * q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
#pragma unroll
        for (int a = 0; a < MS; ++a) {
            const int ro = rr - a;
            if (ro >= 0 && ro < RF) {
#pragma unroll
                for (int b = 0; b < MS; ++b) {
                    const float2 t = reinterpret_cast<const float2*>(kfp)[a * MS + b];
                    const f2_t kk = f2_pack(t.x, t.y);
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        acc2[ro][c] = ffma2(f2_pack(v[c + b], v[c + b]), kk, acc2[ro][c]);
                }
            }
        }
        if constexpr (TNRD_FWD_INTERLEAVE) {
            const int r = rr - 2 * R;   // output row completed by this input row
            if (r >= 1) {
                *reinterpret_cast<float4*>(d0 + (r - 1) * C::PW) = p0;
                *reinterpret_cast<float4*>(d1 + (r - 1) * C::PW) = p1;
            }
            if (r >= 0) {
                p0.x = rbf_cubic_s(f2_lo(acc2[r][0]), tb0, p);
                p0.y = rbf_cubic_s(f2_lo(acc2[r][1]), tb0, p);
                p0.z = rbf_cubic_s(f2_lo(acc2[r][2]), tb0, p);
                p0.w = rbf_cubic_s(f2_lo(acc2[r][3]), tb0, p);
                p1.x = rbf_cubic_s(f2_hi(acc2[r][0]), tb1, p);
                p1.y = rbf_cubic_s(f2_hi(acc2[r][1]), tb1, p);
                p1.z = rbf_cubic_s(f2_hi(acc2[r][2]), tb1, p);
                p1.w = rbf_cubic_s(f2_hi(acc2[r][3]), tb1, p);
            }
        }
    }
    if constexpr (TNRD_FWD_INTERLEAVE) {
        *reinterpret_cast<float4*>(d0 + (RF - 1) * C::PW) = p0;
        *reinterpret_cast<float4*>(d1 + (RF - 1) * C::PW) = p1;
    } else {
        float4 o0[RF], o1[RF];
#pragma unroll
        for (int r = 0; r < RF; ++r) {
            o0[r].x = rbf_cubic_s(f2_lo(acc2[r][0]), tb0, p);
            o0[r].y = rbf_cubic_s(f2_lo(acc2[r][1]), tb0, p);
            o0[r].z = rbf_cubic_s(f2_lo(acc2[r][2]), tb0, p);
            o0[r].w = rbf_cubic_s(f2_lo(acc2[r][3]), tb0, p);
            o1[r].x = rbf_cubic_s(f2_hi(acc2[r][0]), tb1, p);
            o1[r].y = rbf_cubic_s(f2_hi(acc2[r][1]), tb1, p);
            o1[r].z = rbf_cubic_s(f2_hi(acc2[r][2]), tb1, p);
            o1[r].w = rbf_cubic_s(f2_hi(acc2[r][3]), tb1, p);
            if ((r + 1) % BATCH_ROWS == 0 || r == RF - 1) {
#pragma unroll
                for (int q = r - (r % BATCH_ROWS); q <= r; ++q) {
                    *reinterpret_cast<float4*>(d0 + q * C::PW) = o0[q];
                    *reinterpret_cast<float4*>(d1 + q * C::PW) = o1[q];
                }
            }
        }
    }
}

// forward_block with FFMA2 row pairs (pair taps, cubic RBF): rows (2q, 2q+1)
// of the RF x 4 block; an odd last row runs scalar
template <class C, int MS, int RF, int BATCH_ROWS>
__device__ __forceinline__ void forward_block_p2(const StageArgs& p, const float* sU, float* phif,
                                                 const float* kq, uint32_t tb, int blk) {
    constexpr int R = C::R;
    constexpr int NP = RF / 2;
    constexpr bool ODD = (RF & 1) != 0;
    static_assert(NP >= 1, "row pairs need RF >= 2");
    const int by = blk / C::NBX;
    const int bx = blk - by * C::NBX;
    const int x0 = bx * 4, y0 = by * RF;
    TNRD_ASSERT(blk >= 0 && blk < C::NBLK && y0 + RF + 2 * R <= C::UR && x0 + 4 * C::NV <= C::US &&
                y0 + RF <= C::PH && x0 + 4 <= C::PW, 1, blk, C::NBLK);
    f2_t acc2[NP][4];
    float accs[4];
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc2[q][c] = 0ull;
#pragma unroll
    for (int c = 0; c < 4; ++c) accs[c] = 0.0f;
#pragma unroll
    for (int rr = 0; rr < RF + 2 * R; ++rr) {
        float v[4 * C::NV];
        const float* src = sU + (y0 + rr) * C::US + x0;
#pragma unroll
        for (int q = 0; q < C::NV; ++q) {
            const float4 t = lds128(src + 4 * q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int a0 = rr - 2 * q;   // tap row of rot180(k) for output row 2q
            if (a0 >= 1 && a0 <= MS - 1) {
#pragma unroll
                for (int b = 0; b < MS; ++b) {
                    // (kf[a0][b], kf[a0-1][b]) = swap of Q[MS-a0][MS-1-b]
                    const float2 t = qpair<MS>(kq, MS - a0, MS - 1 - b);
                    const f2_t kk = f2_pack(t.y, t.x);
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        acc2[q][c] = ffma2(f2_pack(v[c + b], v[c + b]), kk, acc2[q][c]);
                }
            } else if (a0 == 0 || a0 == MS) {
                // one row of the pair: kf[0][b] (row 2q) or kf[MS-1][b] (row 2q+1)
#pragma unroll
                for (int b = 0; b < MS; ++b) {
                    const float kk = qsingle<MS>(kq, a0 == 0 ? MS - 1 : 0, MS - 1 - b);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        float lo = f2_lo(acc2[q][c]), hi = f2_hi(acc2[q][c]);
                        if (a0 == 0) lo = fmaf(kk, v[c + b], lo);
                        else hi = fmaf(kk, v[c + b], hi);
                        acc2[q][c] = f2_pack(lo, hi);
                    }
                }
            }
        }
        if constexpr (ODD) {
            const int a = rr - (RF - 1);
            if (a >= 0 && a < MS) {
#pragma unroll
                for (int b = 0; b < MS; ++b) {
                    const float kk = qsingle<MS>(kq, MS - 1 - a, MS - 1 - b);
#pragma unroll
                    for (int c = 0; c < 4; ++c) accs[c] = fmaf(kk, v[c + b], accs[c]);
                }
            }
        }
    }
    float acc[RF][4];
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            acc[2 * q][c] = f2_lo(acc2[q][c]);
            acc[2 * q + 1][c] = f2_hi(acc2[q][c]);
        }
    if constexpr (ODD) {
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[RF - 1][c] = accs[c];
    }
    float* dst = phif + y0 * C::PW + x0;
    float4 o[RF];
#pragma unroll
    for (int r = 0; r < RF; ++r) {
        o[r].x = rbf_cubic_s(acc[r][0], tb, p);
        o[r].y = rbf_cubic_s(acc[r][1], tb, p);
        o[r].z = rbf_cubic_s(acc[r][2], tb, p);
        o[r].w = rbf_cubic_s(acc[r][3], tb, p);
        if ((r + 1) % BATCH_ROWS == 0 || r == RF - 1) {
#pragma unroll
            for (int q = r - (r % BATCH_ROWS); q <= r; ++q)
                *reinterpret_cast<float4*>(dst + q * C::PW) = o[q];
        }
    }
}

// Mirrored phi halo without a fix-up pass (EDGE variants of the backward
// filters).  The reference pads phi itself (diffusion.py:180): a phi value
// outside the image is the in-image value at the mirrored position.  When an
// image edge coincides with the tile edge (always on the left / top; on the
// right / bottom when the tile is full) the mirrored positions of a thread's
// RB+2R x 4+2R window lie in the window itself: a window row outside the
// image is READ at its mirrored row (edge_row: region row 2R-1-y above the
// image, 2(TH+R)-1-y below; compile-time row offsets when RB >= R), and after
// a row is loaded its out-of-image columns take the registers of the
// mirrored columns (edge_cols: col c < R <- col 2R-1-c on the left, col
// 4+R+c <- col 4+R-1-c on the right; only the first / last output block of a
// row sees them).  `ef` bits (per thread): 1 left, 2 right, 4 top, 8 bottom
// edge inside this thread's window.  The out-of-image phi cells keep what the
// forward stored there; nobody reads them.  Same values in the same FMA
// order as after the fix_phi pass, so the same bits (tools/ab_outputs.py).
// Ragged right / bottom tiles use fix_phi and the plain variants.
template <class C, int RB>
__device__ __forceinline__ int edge_row(int rr, int oy0, uint32_t ef) {
    constexpr int R = C::R;
    constexpr int TH = C::OBY * RB;
    if constexpr (RB >= R) {
        // out-of-image rows only in the first / last thread row: static remap
        if (rr < R) return oy0 + ((ef & 4u) ? 2 * R - 1 - rr : rr);
        if (rr >= RB + R) return oy0 + ((ef & 8u) ? 2 * (RB + R) - 1 - rr : rr);
        return oy0 + rr;
    } else {
        int row = oy0 + rr;
        if ((ef & 4u) && row < R) row = 2 * R - 1 - row;
        if ((ef & 8u) && row >= TH + R) row = 2 * (TH + R) - 1 - row;
        return row;
    }
}
template <int R, int N>
__device__ __forceinline__ void edge_cols(float (&v)[N], uint32_t ef) {
#pragma unroll
    for (int c = 0; c < R; ++c) {
        v[c] = (ef & 1u) ? v[2 * R - 1 - c] : v[c];
        v[4 + R + c] = (ef & 2u) ? v[4 + R - 1 - c] : v[4 + R + c];
    }
}

// backward_filter with FFMA2 row pairs: force2[q] = rows (2q, 2q+1)
template <class C, int MS, int RB, bool EDGE = false>
__device__ __forceinline__ void backward_filter_p2(const float* ph, const float* kq, int ox0, int oy0,
                                                   f2_t (&force2)[RB / 2][4], uint32_t ef = 0u) {
    constexpr int R = C::R;
    static_assert(RB % 2 == 0, "row pairs");
#pragma unroll
    for (int rr = 0; rr < RB + 2 * R; ++rr) {
        float v[4 * C::NV];
        const int row_ = EDGE ? edge_row<C, RB>(rr, oy0, ef) : oy0 + rr;
        TNRD_ASSERT(row_ >= 0 && row_ < C::PH && ox0 >= 0 && ox0 + 4 * C::NV <= C::PW, 2, row_, C::PH);
        const float* src = ph + row_ * C::PW + ox0;
#pragma unroll
        for (int q = 0; q < C::NV; ++q) {
            const float4 t = lds128(src + 4 * q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
        if constexpr (EDGE) edge_cols<R>(v, ef);
#pragma unroll
        for (int q = 0; q < RB / 2; ++q) {
            const int a0 = rr - 2 * q;   // tap row of k for output row 2q
            if (a0 >= 1 && a0 <= MS - 1) {
#pragma unroll
                for (int b = 0; b < MS; ++b) {
                    const float2 t = qpair<MS>(kq, a0, b);       // (k[a0][b], k[a0-1][b])
                    const f2_t kk = f2_pack(t.x, t.y);
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        force2[q][c] = ffma2(f2_pack(v[c + b], v[c + b]), kk, force2[q][c]);
                }
            } else if (a0 == 0 || a0 == MS) {
#pragma unroll
                for (int b = 0; b < MS; ++b) {
                    const float kk = qsingle<MS>(kq, a0 == 0 ? 0 : MS - 1, b);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        float lo = f2_lo(force2[q][c]), hi = f2_hi(force2[q][c]);
                        if (a0 == 0) lo = fmaf(kk, v[c + b], lo);
                        else hi = fmaf(kk, v[c + b], hi);
                        force2[q][c] = f2_pack(lo, hi);
                    }
                }
            }
        }
    }
}

// forward with the taps in the parameter space: the group's filters one
// after the other over all NT threads, so the filter (and with it the tap
// address) is uniform across every warp
template <class C, int MS, int RF, int F, int NT, bool FAST, int TM, int BATCH_ROWS = RF>
__device__ __forceinline__ void forward_group_pt(const StageArgs& p, const float* sU, float* sPhi,
                                                 const float* kg, const float* tabg, int tid) {
    using TL = TapLayout<MS, C::KP, F, TM>;
    if constexpr (TM >= 2) {
        // both filters per thread: warp-uniform control flow (the uniform
        // datapath is only used outside divergent branches): threads past
        // the last block recompute it and store the same values
        const uint32_t tb0 = static_cast<uint32_t>(__cvta_generic_to_shared(tabg)) + p.tab3_bias;
        const uint32_t tb1 = static_cast<uint32_t>(__cvta_generic_to_shared(tabg + p.tab3_stride)) + p.tab3_bias;
#pragma unroll 1
        for (int b0 = 0; b0 < C::NBLK; b0 += NT)
            forward_block_fp<C, MS, RF, BATCH_ROWS>(p, sU, sPhi, sPhi + C::SPHI, kg, tb0, tb1,
                                                    min(b0 + tid, C::NBLK - 1));
        return;
    } else {
#pragma unroll 1
        for (int fi = 0; fi < F; ++fi) {
            const float* k = kg + fi * TL::per_filter;
            const float* tabf = tabg + fi * p.tab3_stride;
            const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(tabf)) + p.tab3_bias;
            float* phif = sPhi + fi * C::SPHI;
            // warp-uniform control flow (the uniform datapath is only used
            // outside divergent branches): threads past the last block
            // recompute it and store the same values
#pragma unroll 1
            for (int b0 = 0; b0 < C::NBLK; b0 += NT) {
                if constexpr (TM == 1)
                    forward_block_p2<C, MS, RF, BATCH_ROWS>(p, sU, phif, k, tb, min(b0 + tid, C::NBLK - 1));
                else
                    forward_block<C, MS, RF, FAST, BATCH_ROWS, true>(p, sU, phif, k, tb, tabf,
                                                                     min(b0 + tid, C::NBLK - 1));
            }
        }
    }
}

// phi halo outside the image = mirror of in-image phi (the reference pads phi
// itself, diffusion.py:180).  Only the out-of-image band of the phi region is
// rewritten: rows [0, nt) and [h0, PH) and, for the rows in between, columns
// [0, nl) and [w0, PW); sources are in-image.  Ends with a CTA barrier when
// it wrote anything (uniform condition).
template <class C, int F, int NT, int TH, int TW>
__device__ __forceinline__ void fix_phi(const StageArgs& p, float* sPhi, int Y0, int X0,
                                        bool top_halo, bool bot_halo, int tid) {
    constexpr int R = C::R;
    const bool fix_l = X0 - R < 0;
    const bool fix_r = X0 + TW + R > p.W;
    const bool fix_t = !top_halo && (Y0 - R < 0);
    const bool fix_b = !bot_halo && (Y0 + TH + R > p.H);
    if (!(fix_l || fix_r || fix_t || fix_b)) return;
    const int nt_ = fix_t ? min(R, C::PH) : 0;
    const int h0 = fix_b ? max(nt_, min(C::PH, p.H - (Y0 - R))) : C::PH;
    const int nl_ = fix_l ? R : 0;
    const int w0 = fix_r ? max(nl_, min(C::PW, p.W - (X0 - R))) : C::PW;
    const int full_rows = nt_ + (C::PH - h0);
    const int mid_rows = h0 - nt_;
    const int per_f = full_rows * C::PW + mid_rows * (nl_ + C::PW - w0);
    for (int i = tid; i < F * per_f; i += NT) {
        const int j = i / per_f;
        int rem = i - j * per_f;
        int py, px;
        if (rem < full_rows * C::PW) {
            const int rr = rem / C::PW;
            px = rem - rr * C::PW;
            py = rr < nt_ ? rr : h0 + (rr - nt_);
        } else {
            rem -= full_rows * C::PW;
            const int wcols = nl_ + C::PW - w0;
            const int rr = rem / wcols, cc = rem - rr * wcols;
            py = nt_ + rr;
            px = cc < nl_ ? cc : w0 + (cc - nl_);
        }
        const int Y = Y0 - R + py, X = X0 - R + px;
        int sy = Y, sx = X;
        if (X < 0 && X >= -R) sx = -1 - X;
        else if (X >= p.W && X < p.W + R) sx = 2 * p.W - 1 - X;
        if (!top_halo && Y < 0 && Y >= -R) sy = -1 - Y;
        else if (!bot_halo && Y >= p.H && Y < p.H + R) sy = 2 * p.H - 1 - Y;
        if (sy != Y || sx != X) {
            const int spy = sy - (Y0 - R), spx = sx - (X0 - R);
            TNRD_ASSERT(j < F && py >= 0 && py < C::PH && px >= 0 && px < C::PW && spy >= 0 && spy < C::PH &&
                        spx >= 0 && spx < C::PW, 4, spy * C::PW + spx, C::SPHI);
            sPhi[j * C::SPHI + py * C::PW + px] = sPhi[j * C::SPHI + spy * C::PW + spx];
        }
    }
    __syncthreads();
}

// backward of one filter: force += corr(phi_i, k_i) over this thread's
// RB x 4 output block (K: register taps or a parameter-space pointer)
template <class C, int MS, int RB, bool EDGE = false, class K>
__device__ __forceinline__ void backward_filter(const float* ph, const K& k, int ox0, int oy0,
                                                float (&force)[RB][4], uint32_t ef = 0u) {
    constexpr int R = C::R;
#pragma unroll
    for (int rr = 0; rr < RB + 2 * R; ++rr) {
        float v[4 * C::NV];
        const int row_ = EDGE ? edge_row<C, RB>(rr, oy0, ef) : oy0 + rr;
        TNRD_ASSERT(row_ >= 0 && row_ < C::PH && ox0 >= 0 && ox0 + 4 * C::NV <= C::PW, 2, row_, C::PH);
        const float* src = ph + row_ * C::PW + ox0;
#pragma unroll
        for (int q = 0; q < C::NV; ++q) {
            const float4 t = lds128(src + 4 * q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
        if constexpr (EDGE) edge_cols<R>(v, ef);
#pragma unroll
        for (int a = 0; a < MS; ++a) {
            const int ro = rr - a;
            if (ro >= 0 && ro < RB) {
#pragma unroll
                for (int b = 0; b < MS; ++b) {
                    const float kk = k[a * MS + b];
#pragma unroll
                    for (int c = 0; c < 4; ++c) force[ro][c] = fmaf(kk, v[c + b], force[ro][c]);
                }
            }
        }
    }
}

// backward: force += corr(phi_i, k_i) for this thread's filters of the group
template <class C, int MS, int RB, int F, bool EDGE = false>
__device__ __forceinline__ void backward_group(const float* sPhi, const float* tapg, int split,
                                               int ox0, int oy0, float (&force)[RB][4], uint32_t ef = 0u) {
#pragma unroll 1
    for (int fi = split; fi < F; fi += C::NSPLIT) {
        float k[C::KK];
        load_taps<C>(tapg + fi * C::KP, k);
        backward_filter<C, MS, RB, EDGE>(sPhi + fi * C::SPHI, k, ox0, oy0, force, ef);
    }
}

// force accumulators of the parameter-space kernels: FFMA2 row pairs
// (m <= 7) or scalars
template <int MS, int RB, bool P2>
struct ForceAcc {
    f2_t f2[RB / 2 > 0 ? RB / 2 : 1][4];
    float f1[RB][4];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if constexpr (P2) {
                    if (r % 2 == 0) f2[r / 2][c] = 0ull;
                } else {
                    f1[r][c] = 0.0f;
                }
            }
    }
    __device__ __forceinline__ float get(int r, int c) const {
        if constexpr (P2) return (r & 1) ? f2_hi(f2[r >> 1][c]) : f2_lo(f2[r >> 1][c]);
        else return f1[r][c];
    }
};

// backward with parameter-space taps (no filter split: every thread walks
// all of the group's filters, so the tap address is CTA-uniform).  Not
// unrolled (the kernel's hot loop stays within the instruction cache);
// written with pointer increments and a __syncwarp, the form in which ptxas
// keeps the taps in uniform registers (a plain indexed unroll-1 loop loads
// them into per-thread registers with LDC)
template <class C, int MS, int RB, int F, int TM, bool EDGE = false>
__device__ __forceinline__ void backward_group_pt(const float* sPhi, const float* kg, int ox0, int oy0,
                                                  ForceAcc<MS, RB, (TM == 1 || TM == 2)>& acc, uint32_t ef = 0u) {
    static_assert(C::NSPLIT == 1, "parameter-space taps need one thread per output block");
    using TL = TapLayout<MS, C::KP, F, TM>;
    const float* k = kg + TL::bwd0;
    const float* ph = sPhi;
#pragma unroll 1
    for (int fi = 0; fi < F; ++fi, k += TL::per_filter, ph += C::SPHI) {
        if constexpr (TM == 1 || TM == 2) backward_filter_p2<C, MS, RB, EDGE>(ph, k, ox0, oy0, acc.f2, ef);
        else if constexpr (TM == 3) backward_filter<C, MS, RB, EDGE>(ph, FpTap<MS>{k}, ox0, oy0, acc.f1, ef);
        else backward_filter<C, MS, RB, EDGE>(ph, k, ox0, oy0, acc.f1, ef);
        __syncwarp();
    }
}

// sum the filter-split partial forces into the split-0 threads (in split
// order); the others return false.  `red` is free shared memory.
template <class C, int RB>
__device__ __forceinline__ bool reduce_splits(float* red, int split, int obx, int oby,
                                              float (&force)[RB][4]) {
    if (C::NSPLIT == 1) return true;
    __syncthreads();  // everyone is done reading sPhi
    const int slot = (oby * C::OBX + obx) * RB * 4;
    if (split > 0) {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                red[(split - 1) * C::OBX * C::OBY * RB * 4 + slot + r * 4 + c] = force[r][c];
    }
    __syncthreads();
    if (split > 0) return false;
    for (int s2 = 1; s2 < C::NSPLIT; ++s2)
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                force[r][c] += red[(s2 - 1) * C::OBX * C::OBY * RB * 4 + slot + r * 4 + c];
    return true;
}

// epilogue of one pixel: u~ = u - force, reaction, checks, store
__device__ __forceinline__ void finish_pixel(const StageArgs& p, float u, float force,
                                             const float* __restrict__ fin, float* uout,
                                             int64_t off, bool& bad, uint32_t& fbits,
                                             float* fout = nullptr) {
    if (fout) fout[off] = force;
    float res;
    if (p.flags & 0x8u) {
        res = force;
    } else {
        const float fv = __ldg(fin + off);
        if (p.flags & 0x10u) {
            if (!isfinite(fv)) fbits |= 0x1u;
            else if (fv < 0.0f) fbits |= 0x2u;
        }
        res = reaction(u, force, fv, p);
    }
    if (!isfinite(res)) bad = true;
    uout[off] = res;
}

// finish_pixel with the observation already loaded
__device__ __forceinline__ void finish_pixel_f(const StageArgs& p, float u, float force, float fv,
                                               float* uout, int64_t off, bool& bad, uint32_t& fbits,
                                               float* fout = nullptr) {
    if (fout) fout[off] = force;
    float res;
    if (p.flags & 0x8u) {
        res = force;
    } else {
        if (p.flags & 0x10u) {
            if (!isfinite(fv)) fbits |= 0x1u;
            else if (fv < 0.0f) fbits |= 0x2u;
        }
        res = reaction(u, force, fv, p);
    }
    if (!isfinite(res)) bad = true;
    uout[off] = res;
}

// programmatic dependent launch: wait for the predecessor grid's completion
// (and memory) / let the successor grid be scheduled
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void report(const StageArgs& p, bool bad, uint32_t fbits) {
    if (bad) atomicMin(p.status, (uint32_t)p.stage);
    if (fbits) atomicAnd(p.status + 1, ~fbits);
}


// ---- RBF tables by bulk copy (TMA engine) ----------------------------------
// The parameter-space-taps kernels fetch a group's RBF tables with one
// cp.async.bulk issued by one thread and completed on an mbarrier: no
// per-thread copy loop in the group loop (which makes ptxas keep the group
// index, and with it the tap addresses, out of the uniform datapath).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread: dst[0, n) <- src[0, n) (16-byte aligned, n % 4 == 0), completing on bar
__device__ __forceinline__ void tbar_fetch(float* dst, const float* src, int n, uint64_t* bar) {
    const uint32_t bytes = 4u * (uint32_t)n;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the generic reads of dst
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
// bounded wait: a lost completion traps instead of hanging the GPU
__device__ __forceinline__ void tbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    for (uint32_t spin = 0;; ++spin) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) return;
        if (spin > (1u << 26)) __trap();
    }
}


// ---- thread-block clusters (one launch per stage on small grids) ----------
// stage_kernel_cl / stage_kernel_cl_pt run a tile's filter groups on the CTAs
// of one cluster (rank r takes the r-th of cluster-size contiguous, balanced
// group ranges), leave each CTA's partial force in its shared memory and sum
// the partials IN RANK ORDER through distributed shared memory, each CTA
// finishing 1 / cluster-size of the tile's pixels.
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 128-bit load of the shared-memory word at `addr` (a shared::cta address of
// this CTA's window) in the CTA of cluster rank `rank`
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(addr), "r"(rank));
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(ra)
                 : "memory");
    return v;
}
constexpr int kMaxCluster = 8;   // portable cluster size limit

// ---- tile kernel: one CTA = one output tile, all filter groups -------------
// PT: taps read from the parameter space (`kp` = this stage's TapBlock)
// instead of being staged in shared memory and held in registers
// mirrored phi halo inside the backward's window instead of the fix_phi pass
// (tile and cluster kernels; 0 = always fix_phi, for A/B runs)
#ifndef TNRD_EDGE_BACKWARD
#define TNRD_EDGE_BACKWARD 1
#endif

#ifdef TNRD_PHASE_TRACE
// per-phase CTA clock totals of the tile kernel (tools/phase_trace.py):
// 0 staging, 1 forward + RBF, 2 phi fix-up + table fetch, 3 backward (to the
// next group's barrier), 4 epilogue, 5 CTAs
__device__ unsigned long long g_phase[8];
#define TNRD_PHASE_MARK(i)                                                     \
    if (tid == 0) {                                                            \
        const long long t_ = clock64();                                        \
        atomicAdd(&g_phase[i], (unsigned long long)(t_ - ph_t));               \
        ph_t = t_;                                                             \
    }
#else
#define TNRD_PHASE_MARK(i)
#endif

// CLU: launched as clusters along x; the cluster's CTAs share one tile (see
// the cluster helpers above)
template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, bool PT, int TM = 0, bool CLU = false>
__device__ __forceinline__ void stage_tile_body(const StageArgs& p, const float* kp) {
    using C = StageCfg<MS, TH, TW, RF, RB, NT, F>;
    constexpr int R = C::R;
    extern __shared__ __align__(16) float smem[];
    float* sU = smem;
    float* sPhi = sU + C::SU;
    // PT: no tap buffer, one (cubic) table buffer: u | phi[F] | tab3[F]
    float* sTap = sPhi + F * C::SPHI;
    float* sTab = PT ? sTap : sTap + 2 * F * C::KP;
    const int tabsz = F * (PT ? p.tab3_stride : p.tab_stride);

    const int tid = threadIdx.x;
    const int img = blockIdx.z;
    // Cluster launches: grid (cluster, tiles, batch), the cluster along x, so
    // the rank is blockIdx.x and this CTA's group range -- the rank-th of
    // `cluster` contiguous ranges, the first cl_gextra one group longer --
    // needs no division.  (With %cluster_ctarank, or a division by the
    // cluster size, ptxas computed the group index outside the uniform
    // datapath in some instantiations -- m = 9, m = 3 -- and the taps fell
    // back to per-thread LDC; SASS checked.)
    const int cln = CLU ? p.cluster : 1;
    const int clr = CLU ? (int)blockIdx.x : 0;
    const int tile_y = CLU ? (int)blockIdx.y / p.cl_tiles_x : (int)blockIdx.y;
    const int tile_x = CLU ? (int)blockIdx.y - tile_y * p.cl_tiles_x : (int)blockIdx.x;
    const int Y0 = tile_y * TH;
    const int X0 = tile_x * TW;
    const int gbeg = CLU ? clr * p.cl_gper + min(clr, p.cl_gextra) : 0;
    const int gend = CLU ? gbeg + p.cl_gper + (clr < p.cl_gextra ? 1 : 0) : p.ngroups;
    const float* __restrict__ uin = p.u_in + (int64_t)img * p.img_stride;
    const float* __restrict__ fin = p.f + (int64_t)img * p.img_stride;
    float* __restrict__ uout = p.u_out + (int64_t)img * p.img_stride;
    float* fout = p.force_out ? p.force_out + (int64_t)img * p.img_stride : nullptr;
    const bool top_halo = p.flags & 0x2u;
    const bool bot_halo = p.flags & 0x4u;

    __shared__ __align__(8) uint64_t tbar;  // PT: the table buffer's fills
    if constexpr (PT) {
        if (tid == 0) {
            tbar_init(&tbar);
            if (gbeg < gend) tbar_fetch(sTab, p.tab3 + (size_t)gbeg * tabsz, tabsz, &tbar);
        }
        __syncthreads();  // barrier initialised before anyone waits
    } else {
        if (gbeg < gend) prefetch_group<C, F, NT>(p, sTap, sTab, gbeg, 0, tid);
    }
    pdl_wait();     // the previous stage wrote u_in
    pdl_trigger();
#ifdef TNRD_PHASE_TRACE
    long long ph_t = clock64();
    if (tid == 0) atomicAdd(&g_phase[5], 1ull);
#endif
    stage_u_tile<C, NT>(p, sU, uin, Y0, X0, top_halo, bot_halo, tid);

    const int split = PT ? 0 : tid / (C::OBX * C::OBY);  // which filters of a group
    const int obx = tid % C::OBX, oby = (tid / C::OBX) % C::OBY;
    const int ox0 = obx * 4, oy0 = oby * RB;
    // image edges in this tile's phi region: when they coincide with the
    // tile's edges the backward mirrors phi inside its own window (EDGE
    // variants: edge_row / edge_cols, no fix-up pass); ragged right / bottom
    // tiles run fix_phi
    uint32_t ef = 0u;
    bool edge_static = false;
    if constexpr (TNRD_EDGE_BACKWARD) {
        const bool fix_l = X0 - R < 0, fix_r = X0 + TW + R > p.W;
        const bool fix_t = !top_halo && Y0 - R < 0, fix_b = !bot_halo && Y0 + TH + R > p.H;
        edge_static = (fix_l || fix_r || fix_t || fix_b) && (!fix_r || p.W - X0 == TW) &&
                      (!fix_b || p.H - Y0 == TH);
        if (edge_static)
            ef = (fix_l && obx == 0 ? 1u : 0u) | (fix_r && obx == C::OBX - 1 ? 2u : 0u) |
                 (fix_t && oy0 < R ? 4u : 0u) | (fix_b && oy0 + RB + R > TH ? 8u : 0u);
    }
    constexpr int GS = TapLayout<MS, C::KP, F, TM>::group;   // PT tap floats per filter group
    float force[RB][4];
    ForceAcc<MS, RB, (TM == 1 || TM == 2)> facc;   // PT: FFMA2 row pairs (TM 1, 2) or scalars
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) force[r][c] = 0.0f;
    if constexpr (PT) facc.zero();

    for (int g = gbeg; g < gend; ++g) {
        const int buf = PT ? 0 : (g - gbeg) & 1;
        if constexpr (PT) tbar_wait(&tbar, (g - gbeg) & 1);  // fill g - gbeg of the one buffer
        else cp_async_wait_all();
        __syncthreads();  // params of group g landed; previous bwd done with sPhi
        TNRD_PHASE_MARK(g == gbeg ? 0 : 3)
        if constexpr (!PT)
            if (g + 1 < gend) prefetch_group<C, F, NT>(p, sTap, sTab, g + 1, buf ^ 1, tid);
        const float* tapg = PT ? kp + g * GS : sTap + buf * F * C::KP;
        const float* tabg = sTab + buf * tabsz;
        if constexpr (PT) forward_group_pt<C, MS, RF, F, NT, FAST, TM>(p, sU, sPhi, tapg, tabg, tid);
        else forward_group<C, MS, RF, F, FAST>(p, sU, sPhi, tapg, tabg, tid);
        __syncthreads();
        TNRD_PHASE_MARK(1)
        // PT: the table is free -- fetch the next group's under fix-up + backward
        if constexpr (PT)
            if (tid == 0 && g + 1 < gend) tbar_fetch(sTab, p.tab3 + (size_t)(g + 1) * tabsz, tabsz, &tbar);
#ifdef TNRD_PROBE_NO_BACKWARD
        // perf probe only (wrong results): the stage without its adjoint
        // convolution = the ceiling of any tensor-core offload of the backward
        if (p.H > 0) continue;
#endif
        if (edge_static) {
            TNRD_PHASE_MARK(2)
            if constexpr (PT) backward_group_pt<C, MS, RB, F, TM, true>(sPhi, tapg, ox0, oy0, facc, ef);
            else backward_group<C, MS, RB, F, true>(sPhi, tapg, split, ox0, oy0, force, ef);
        } else {
            fix_phi<C, F, NT, TH, TW>(p, sPhi, Y0, X0, top_halo, bot_halo, tid);
            TNRD_PHASE_MARK(2)
            if constexpr (PT) backward_group_pt<C, MS, RB, F, TM>(sPhi, tapg, ox0, oy0, facc);
            else backward_group<C, MS, RB, F>(sPhi, tapg, split, ox0, oy0, force);
        }
    }
    if constexpr (PT) {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) force[r][c] = facc.get(r, c);
    }
#ifdef TNRD_PHASE_TRACE
    __syncthreads();
    TNRD_PHASE_MARK(3)
#endif
    if constexpr (CLU) {
        // partial force of this CTA's groups -> shared memory (past the
        // scratch of reduce_splits), then the ordered sum over the cluster
        constexpr int TPX = TH * TW;
        static_assert(C::NSPLIT * TPX <= F * C::SPHI, "partial force must fit the phi buffers");
        static_assert(TW % 4 == 0 && (C::SPHI % 4) == 0, "float4 partials");
        const bool full = reduce_splits<C, RB>(sPhi, split, obx, oby, force);
        if (C::NSPLIT == 1) __syncthreads();   // everyone is done reading sPhi
        float* sPart = sPhi + (C::NSPLIT - 1) * TPX;
        if (full) {
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                TNRD_ASSERT((oy0 + r) * TW + ox0 + 4 <= TPX, 8, (oy0 + r) * TW + ox0, TPX);
                *reinterpret_cast<float4*>(sPart + (oy0 + r) * TW + ox0) =
                    make_float4(force[r][0], force[r][1], force[r][2], force[r][3]);
            }
        }
        cluster_sync_all();   // every CTA's partial is visible cluster-wide
        constexpr int QUADS = TPX / 4;
        const int qs = (QUADS + cln - 1) / cln;
        const int qend = min(QUADS, (clr + 1) * qs);
        const uint32_t pa = smem_addr(sPart);
        bool bad = false;
        uint32_t fbits = 0;
        for (int q = clr * qs + tid; q < qend; q += NT) {
            const int y = (4 * q) / TW, x = (4 * q) % TW;
            TNRD_ASSERT(q >= 0 && q < QUADS && y < TH && (y + 2 * R) * C::US + x + 3 + 2 * R < C::SU, 8, q, QUADS);
            float4 v[kMaxCluster];
#pragma unroll
            for (int r = 0; r < kMaxCluster; ++r)
                if (r < cln) v[r] = ld_cluster_f4(pa + 16u * (uint32_t)q, (uint32_t)r);
            float4 acc = v[0];
#pragma unroll
            for (int r = 1; r < kMaxCluster; ++r)
                if (r < cln) { acc.x += v[r].x; acc.y += v[r].y; acc.z += v[r].z; acc.w += v[r].w; }
            const int Y = Y0 + y;
            if (Y >= p.H) continue;
            const float fa[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int X = X0 + x + c;
                if (X >= p.W) continue;
                finish_pixel(p, sU[(y + 2 * R) * C::US + x + c + 2 * R], fa[c], fin, uout,
                             (int64_t)Y * p.ld + X, bad, fbits, fout);
            }
        }
        report(p, bad, fbits);
        cluster_sync_all();   // no CTA leaves while a peer may still read its partial
        TNRD_PHASE_MARK(4)
        return;
    }
    if (!reduce_splits<C, RB>(sPhi, split, obx, oby, force)) return;

    bool bad = false;
    uint32_t fbits = 0;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int Y = Y0 + oy0 + r;
        if (Y >= p.H) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int X = X0 + ox0 + c;
            if (X >= p.W) continue;
            finish_pixel(p, sU[(oy0 + r + 2 * R) * C::US + ox0 + c + 2 * R], force[r][c], fin, uout,
                         (int64_t)Y * p.ld + X, bad, fbits, fout);
        }
    }
    report(p, bad, fbits);
    TNRD_PHASE_MARK(4)
}

template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, int MINB>
__global__ void __launch_bounds__(NT, MINB) stage_kernel(const StageArgs p) {
    stage_tile_body<MS, TH, TW, RF, RB, NT, FAST, F, false>(p, nullptr);
}

// taps of one stage in the kernel parameter space (<= 32 KB of parameters
// on sm_100): read with warp-uniform addresses by the uniform datapath, they
// cost no shared-memory traffic and no per-thread registers
constexpr int kMaxParamTaps = 7680;
template <int N>
struct TapBlock {
    static_assert(N <= kMaxParamTaps, "kernel parameters are limited to 32 KB");
    float k[N];
};

template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, int MINB, class TB, int TM>
__global__ void __launch_bounds__(NT, MINB) stage_kernel_pt(const StageArgs p, const __grid_constant__ TB tk) {
    stage_tile_body<MS, TH, TW, RF, RB, NT, FAST, F, true, TM>(p, tk.k);
}

// cluster variants (launched with a cluster dimension of 2..8 CTAs along x;
// grid.x = tiles_x * cluster size): one launch per stage on grids that are
// too small to fill the SMs with whole-tile CTAs
template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, int MINB>
__global__ void __launch_bounds__(NT, MINB) stage_kernel_cl(const StageArgs p) {
    stage_tile_body<MS, TH, TW, RF, RB, NT, FAST, F, false, 0, true>(p, nullptr);
}
template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, int MINB, class TB, int TM>
__global__ void __launch_bounds__(NT, MINB) stage_kernel_cl_pt(const StageArgs p, const __grid_constant__ TB tk) {
    stage_tile_body<MS, TH, TW, RF, RB, NT, FAST, F, true, TM, true>(p, tk.k);
}

// ---- split kernels: work units = (tile, filter group) ----------------------
//
// For grids too small to fill 148 SMs with whole tiles (a single 512^2 image
// has 64 large / 256 small tiles) a stage runs as two launches:
//
//   stage_kernel_split  a persistent grid of (SMs x resident CTAs) computes
//       (tile, filter group) units: one group's partial force over one tile,
//       stored to the workspace.  CTA c takes the c-th of gridDim.x
//       contiguous, balanced ranges of the tile-major unit sequence (the u
//       tile is staged once per tile the range touches).
//   stage_reduce_kernel  sums each pixel's ngroups partials IN GROUP ORDER
//       and runs the epilogue, over all SMs.
//
// The summation order is fixed by the unit structure, not by which CTA ran
// what, so results are bit-reproducible and identical for any grid (strips
// == whole image).  No state survives a launch.
#ifndef TNRD_SPLIT_RBF_ROWS
#define TNRD_SPLIT_RBF_ROWS 1   // phi rows per store batch in the split kernel's forward
#endif
struct SplitWs {
    float* part;       // [tiles][ngroups][TH*TW] partial forces
    int tiles_x, tiles_y, tiles;
    // SM-aware range assignment of the parameter-space split kernel (0 = off:
    // CTA c takes range c).  With the grid = map_sms x P resident CTAs, the
    // k-th CTA to arrive on SM s (k < P) takes range k * map_sms + s, so
    // the ranges that carry one extra unit (the first units % grid) land on
    // distinct SMs; measured on B200 the block scheduler otherwise pairs two
    // of them on one SM (12 units there instead of 11).  Ranges are claimed
    // with a CAS on `ctl`, and a CTA that arrives as a third on its SM (the
    // SMs were shared with another kernel) takes any unclaimed range, so
    // every range runs exactly once whatever the placement.  The last CTA to
    // finish zeroes `ctl` for the next launch on this workspace.
    uint32_t* ctl;     // [kSplitCtlSms] per-SM arrivals | [kSplitCtlRanges] claimed | count | done
    int map_sms;
};
constexpr int kSplitCtlSms = 256;
constexpr int kSplitCtlRanges = 4096;
constexpr size_t kSplitCtlWords = kSplitCtlSms + kSplitCtlRanges + 2;

// thread 0: claim an unclaimed range (lowest first); -1 when all are taken
__device__ __forceinline__ int split_claim_any(const SplitWs& ws) {
    uint32_t* claimed = ws.ctl + kSplitCtlSms;
    uint32_t* count = claimed + kSplitCtlRanges;
    for (int c = 0; c < (int)gridDim.x; ++c) {
        if (atomicAdd(count, 0u) >= gridDim.x) return -1;
        if (atomicCAS(claimed + c, 0u, 1u) == 0u) {
            atomicAdd(count, 1u);
            return c;
        }
    }
    return -1;
}
// thread 0: this CTA's first range (SM-aware when ws.map_sms > 0)
__device__ __forceinline__ int split_claim_first(const SplitWs& ws) {
    if (ws.map_sms <= 0) return blockIdx.x;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if ((int)smid < ws.map_sms && (int)smid < kSplitCtlSms) {
        const uint32_t k = atomicAdd(ws.ctl + smid, 1u);
        const uint32_t P = gridDim.x / (uint32_t)ws.map_sms;
        // the LAST CTA to arrive on an SM takes the lowest range (the ranges
        // with the extra unit): its warps have the higher slots, which the
        // warp arbiter issues first (measured: the earlier CTA of an SM
        // finishes its share later)
        const int c = (int)(P - 1 - k) * ws.map_sms + (int)smid;
        if (k < P && c < (int)gridDim.x && atomicCAS(ws.ctl + kSplitCtlSms + c, 0u, 1u) == 0u) {
            atomicAdd(ws.ctl + kSplitCtlSms + kSplitCtlRanges, 1u);
            return c;
        }
    }
    return split_claim_any(ws);
}
// thread 0, after the CTA's last range: the last CTA of the launch resets ctl
__device__ __forceinline__ void split_finish(const SplitWs& ws) {
    if (ws.map_sms <= 0) return;
    __threadfence();
    uint32_t* done = ws.ctl + kSplitCtlSms + kSplitCtlRanges + 1;
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
        __threadfence();
        for (int i = 0; i < kSplitCtlSms; ++i) ws.ctl[i] = 0u;
        for (int i = 0; i < (int)gridDim.x && i < kSplitCtlRanges; ++i) ws.ctl[kSplitCtlSms + i] = 0u;
        ws.ctl[kSplitCtlSms + kSplitCtlRanges] = 0u;
        *done = 0u;
        __threadfence();
    }
}

#ifdef TNRD_SPLIT_TRACE
// per-CTA timeline for tools/split_trace.py: smid, t0, t1, units | first << 32
__device__ unsigned long long g_split_trace[4096][4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F>
__device__ __forceinline__ void stage_split_body(const StageArgs& p, const SplitWs& ws) {
#ifdef TNRD_SPLIT_TRACE
    const unsigned long long tr_t0 = gtimer();
#endif
    using C = StageCfg<MS, TH, TW, RF, RB, NT, F>;
    constexpr int TPX = TH * TW;
    extern __shared__ __align__(16) float smem[];
    float* sU = smem;
    float* sPhi = sU + C::SU;
    float* sTap = sPhi + F * C::SPHI;
    float* sTab = sTap + 2 * F * C::KP;
    const int tabsz = F * p.tab_stride;
    const int tid = threadIdx.x;
    const int ng = p.ngroups;
    const bool top_halo = p.flags & 0x2u;
    const bool bot_halo = p.flags & 0x4u;

    const int units = ws.tiles * ng;
    const int nb = units / (int)gridDim.x, extra = units % (int)gridDim.x;
    const int c = blockIdx.x;
    const int ubeg = c * nb + min(c, extra);
    const int uend = ubeg + nb + (c < extra ? 1 : 0);

    const int split = tid / (C::OBX * C::OBY);
    const int obx = tid % C::OBX, oby = (tid / C::OBX) % C::OBY;
    const int ox0 = obx * 4, oy0 = oby * RB;

    if (ubeg < uend) prefetch_group<C, F, NT>(p, sTap, sTab, ubeg % ng, 0, tid);
    pdl_wait();     // the previous stage wrote u_in
    pdl_trigger();  // the reduction may be scheduled as CTAs retire
    int buf = 0, cur_tile = -1;
    for (int unit = ubeg; unit < uend; ++unit) {
        const int tile = unit / ng, g = unit - tile * ng;
        const int img = tile / (ws.tiles_x * ws.tiles_y);
        const int trem = tile - img * (ws.tiles_x * ws.tiles_y);
        const int Y0 = (trem / ws.tiles_x) * TH, X0 = (trem % ws.tiles_x) * TW;
        if (tile != cur_tile) {
            __syncthreads();  // the previous unit is done with sU
            stage_u_tile<C, NT>(p, sU, p.u_in + (int64_t)img * p.img_stride, Y0, X0, top_halo,
                                bot_halo, tid);
            cur_tile = tile;
        }
        cp_async_wait_all();
        __syncthreads();  // params + u tile in smem; previous unit done with sPhi
        if (unit + 1 < uend) prefetch_group<C, F, NT>(p, sTap, sTab, (unit + 1) % ng, buf ^ 1, tid);
        const float* tapg = sTap + buf * F * C::KP;
        const float* tabg = sTab + buf * tabsz;
        forward_group<C, MS, RF, F, FAST, TNRD_SPLIT_RBF_ROWS>(p, sU, sPhi, tapg, tabg, tid);
        __syncthreads();
        fix_phi<C, F, NT, TH, TW>(p, sPhi, Y0, X0, top_halo, bot_halo, tid);
        float force[RB][4];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) force[r][cc] = 0.0f;
        backward_group<C, MS, RB, F>(sPhi, tapg, split, ox0, oy0, force);
        if (reduce_splits<C, RB>(sPhi, split, obx, oby, force)) {
            float* dst = ws.part + ((size_t)tile * ng + g) * TPX + oy0 * TW + ox0;
#pragma unroll
            for (int r = 0; r < RB; ++r)
                __stcg(reinterpret_cast<float4*>(dst + r * TW),
                       make_float4(force[r][0], force[r][1], force[r][2], force[r][3]));
        }
        buf ^= 1;
    }
#ifdef TNRD_SPLIT_TRACE
    if (tid == 0 && blockIdx.x < 4096) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_split_trace[blockIdx.x][0] = smid;
        g_split_trace[blockIdx.x][1] = tr_t0;
        g_split_trace[blockIdx.x][2] = gtimer();
        g_split_trace[blockIdx.x][3] = (unsigned long long)(uend - ubeg) | ((unsigned long long)(unsigned)ubeg << 32);
    }
#endif
}

// split kernel with parameter-space taps: the same units and summation
// order, walked as tile segments (u staged in the outer loop) so that the
// inner group loop holds only shared-memory traffic and the partial store:
// ptxas then keeps the group index -- and the tap addresses -- uniform.
template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, int TM>
__device__ __forceinline__ void stage_split_body_pt(const StageArgs& p, const SplitWs& ws, const float* kp) {
    using C = StageCfg<MS, TH, TW, RF, RB, NT, F>;
    constexpr int TPX = TH * TW;
    extern __shared__ __align__(16) float smem[];
    float* sU = smem;
    float* sPhi = sU + C::SU;
    float* sTab = sPhi + F * C::SPHI;   // one cubic table buffer
    const int tabsz = F * p.tab3_stride;
    const int tid = threadIdx.x;
    const int ng = p.ngroups;
    const bool top_halo = p.flags & 0x2u;
    const bool bot_halo = p.flags & 0x4u;

    const int units = ws.tiles * ng;
    const int nb = units / (int)gridDim.x, extra = units % (int)gridDim.x;
    const int obx = tid % C::OBX, oby = tid / C::OBX;
    const int ox0 = obx * 4, oy0 = oby * RB;

    __shared__ __align__(8) uint64_t tbar;  // the table buffer's fills
    __shared__ int s_range;                 // range being processed (-1: none left)
    if (tid == 0) {
        tbar_init(&tbar);
        // the ranges' control words are not written by the previous grid,
        // so the claim may run before the dependency wait
        const int c = split_claim_first(ws);
        s_range = c;
        if (c >= 0 && nb + (c < extra ? 1 : 0) > 0)
            tbar_fetch(sTab, p.tab3 + (size_t)((c * nb + min(c, extra)) % ng) * tabsz, tabsz, &tbar);
    }
    __syncthreads();  // barrier initialised before anyone waits
    pdl_wait();       // the previous stage wrote u_in
    pdl_trigger();    // the reduction may be scheduled as CTAs retire
#ifdef TNRD_SPLIT_TRACE
    const unsigned long long tr_t0 = gtimer();
    int ubeg = 0, nunits = 0;
#endif
    uint32_t fills = 0;   // table fills consumed before this range (mbarrier parity)
  for (;;) {
    const int c = s_range;
    if (c < 0) break;
#ifndef TNRD_SPLIT_TRACE
    const int ubeg = c * nb + min(c, extra);
    const int nunits = nb + (c < extra ? 1 : 0);
#else
    ubeg = c * nb + min(c, extra);
    nunits = nb + (c < extra ? 1 : 0);
#endif
    int k = 0;        // units done in this range (= table fills completed)
    while (k < nunits) {
        const int unit = ubeg + k;
        const int tile = unit / ng, g0 = unit - tile * ng;
        const int gend = min(ng, g0 + (nunits - k));
        const int img = tile / (ws.tiles_x * ws.tiles_y);
        const int trem = tile - img * (ws.tiles_x * ws.tiles_y);
        const int Y0 = (trem / ws.tiles_x) * TH, X0 = (trem % ws.tiles_x) * TW;
        __syncthreads();  // the previous unit is done with sU
        stage_u_tile<C, NT>(p, sU, p.u_in + (int64_t)img * p.img_stride, Y0, X0, top_halo, bot_halo, tid);
        float* dst = ws.part + (size_t)tile * ng * TPX + oy0 * TW + ox0;
        for (int g = g0; g < gend; ++g, ++k) {
            tbar_wait(&tbar, (fills + k) & 1);
            __syncthreads();  // table + u tile in smem; previous unit done with sPhi
            const float* tapg = kp + g * TapLayout<MS, C::KP, F, TM>::group;
            const float* tabg = sTab;
            // all RF rows' table lookups before the phi stores (with the taps
            // out of the registers this pays here too: +1% C2 on B200)
            forward_group_pt<C, MS, RF, F, NT, FAST, TM>(p, sU, sPhi, tapg, tabg, tid);
            __syncthreads();
            // the table is free: fetch the next unit's under fix-up + backward
            if (tid == 0 && k + 1 < nunits)
                tbar_fetch(sTab, p.tab3 + (size_t)(g + 1 < ng ? g + 1 : 0) * tabsz, tabsz, &tbar);
            fix_phi<C, F, NT, TH, TW>(p, sPhi, Y0, X0, top_halo, bot_halo, tid);
            ForceAcc<MS, RB, (TM == 1 || TM == 2)> facc;
            facc.zero();
            backward_group_pt<C, MS, RB, F, TM>(sPhi, tapg, ox0, oy0, facc);
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                TNRD_ASSERT(tile < ws.tiles && g < ng && oy0 * TW + ox0 + r * TW + 4 <= TPX, 7, tile, ws.tiles);
                __stcg(reinterpret_cast<float4*>(dst + (size_t)g * TPX + r * TW),
                       make_float4(facc.get(r, 0), facc.get(r, 1), facc.get(r, 2), facc.get(r, 3)));
            }
        }
    }
    fills += nunits;
    __syncthreads();  // every thread has read s_range and is done with sTab
    if (tid == 0) {
        const int c2 = ws.map_sms > 0 ? split_claim_any(ws) : -1;
        s_range = c2;
        if (c2 >= 0 && nb + (c2 < extra ? 1 : 0) > 0)
            tbar_fetch(sTab, p.tab3 + (size_t)((c2 * nb + min(c2, extra)) % ng) * tabsz, tabsz, &tbar);
    }
    __syncthreads();
  }
    if (tid == 0) split_finish(ws);
#ifdef TNRD_SPLIT_TRACE
    if (tid == 0 && blockIdx.x < 4096) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_split_trace[blockIdx.x][0] = smid;
        g_split_trace[blockIdx.x][1] = tr_t0;
        g_split_trace[blockIdx.x][2] = gtimer();
        g_split_trace[blockIdx.x][3] = (unsigned long long)nunits | ((unsigned long long)(unsigned)ubeg << 32);
    }
#endif
}

template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, int MINB>
__global__ void __launch_bounds__(NT, MINB) stage_kernel_split(const StageArgs p, const SplitWs ws) {
    stage_split_body<MS, TH, TW, RF, RB, NT, FAST, F>(p, ws);
}

template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, int MINB, class TB, int TM>
__global__ void __launch_bounds__(NT, MINB) stage_kernel_split_pt(const StageArgs p, const SplitWs ws,
                                                                 const __grid_constant__ TB tk) {
    stage_split_body_pt<MS, TH, TW, RF, RB, NT, FAST, F, TM>(p, ws, tk.k);
}

// sum of a pixel quad's partials in group order, then the epilogue (u from
// u_in, floored on the first stage exactly as the tile kernels stage it).
// Up to 24 groups all partial loads of a quad are in flight at once, with
// the quad's u and f loads.
#ifndef TNRD_REDUCE_NV
#define TNRD_REDUCE_NV 24
#endif
template <int TH, int TW>
__global__ void __launch_bounds__(128) stage_reduce_kernel(const StageArgs p, const SplitWs ws) {
    constexpr int TPX = TH * TW;
    constexpr int NV = TNRD_REDUCE_NV;
    const int ng = p.ngroups;
    const int64_t quads = (int64_t)ws.tiles * (TPX / 4);
    bool bad = false;
    uint32_t fbits = 0;
    pdl_wait();     // all partials written
    pdl_trigger();
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < quads;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int tile = (int)(q / (TPX / 4));
        const int i = 4 * (int)(q - (int64_t)tile * (TPX / 4));
        const int img = tile / (ws.tiles_x * ws.tiles_y);
        const int trem = tile - img * (ws.tiles_x * ws.tiles_y);
        const int Y = (trem / ws.tiles_x) * TH + i / TW;
        const int Xq = (trem % ws.tiles_x) * TW + i % TW;
        if (Y >= p.H) continue;
        const float* __restrict__ uin = p.u_in + (int64_t)img * p.img_stride;
        const float* __restrict__ fin = p.f + (int64_t)img * p.img_stride;
        float* __restrict__ uout = p.u_out + (int64_t)img * p.img_stride;
        float* fout = p.force_out ? p.force_out + (int64_t)img * p.img_stride : nullptr;
        float uq[4], fq[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int64_t off = (int64_t)Y * p.ld + min(Xq + c, p.W - 1);
            uq[c] = __ldg(uin + off);
            fq[c] = __ldg(fin + off);
        }
        const float* src = ws.part + (size_t)tile * ng * TPX + i;
        // batches of NV partial loads in flight, summed in group order
        float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        for (int g0 = 0; g0 < ng; g0 += NV) {
            float4 v[NV];
#pragma unroll
            for (int g = 0; g < NV; ++g)
                if (g0 + g < ng) v[g] = __ldcg(reinterpret_cast<const float4*>(src + (size_t)(g0 + g) * TPX));
#pragma unroll
            for (int g = 0; g < NV; ++g)
                if (g0 + g < ng) {
                    if (g0 + g == 0) {
                        acc = v[0];
                    } else {
                        acc.x += v[g].x; acc.y += v[g].y; acc.z += v[g].z; acc.w += v[g].w;
                    }
                }
        }
        const float fa[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int X = Xq + c;
            if (X >= p.W) continue;
            float u = uq[c];
            if (p.flags & 0x1u) u = fmaxf(u, p.u0_floor);
            finish_pixel_f(p, u, fa[c], fq[c], uout, (int64_t)Y * p.ld + X, bad, fbits, fout);
        }
    }
    report(p, bad, fbits);
}

}  // namespace tnrd

// tnrd_stage_tc.cuh -- fused TNRD stage with the forward filter bank on the
// 5th-generation tensor cores (tcgen05.mma kind::tf32, 3xTF32 split).
//
// Same stage operator as tnrd_stage.cuh (reference diffusion.py:184-194);
// only the forward convolution z_i = conv2d(u, k_i) (imageops.py:53-72)
// moves from FFMA to tcgen05:
//
//   * the 49-tap stencil is a GEMM D[points x 16 filters] = A[points x taps]
//     B[taps x 16 filters] per batch of 16 filters.  No im2col: for tap row a
//     and point class o = x mod 4, the A rows of the 8 class-o points of one
//     image row are the overlapping 32-byte windows u[y+a][4k+o .. 4k+o+7]
//     of a class-shifted copy of the u row, i.e. exactly a K-major
//     SWIZZLE_NONE core matrix with rows 16 B apart (LBO = 16 B: the second
//     K-chunk starts one window later; SBO = the copy's row stride).  One
//     M=128 MMA covers 16 image rows x 8 class-o points of the 32-column phi
//     region; a 32 x 32 region = 2 bands x 4 classes = 8 MMA blocks.
//     (MN-major tf32 B operands, which would let one copy serve all classes,
//     produced all-zero accumulators on this B200/driver in
//     tools/probes/mma_mn_probe.cu, so the classes are separate copies.)
//   * 3xTF32: u = u_hi + u_lo, k = k_hi + k_lo (hi = cvt.rna.tf32), D +=
//     hi*hi + lo*hi + hi*lo with fp32 accumulation in TMEM (~2^-21 relative,
//     single-pass TF32 fails the 1e-4 bar, 3xTF32 passes).
//   * accumulators live in TMEM (2 x 128 columns, double-buffered by batch
//     so the tensor core computes batch b+1 while the CUDA cores run the RBF
//     + backward pass of batch b, 4 filters at a time); commit -> mbarrier ->
//     tcgen05.ld.  109 KB of shared memory and 256 TMEM columns per CTA: two
//     CTAs per SM.
//   * RBF, phi mirror fix-up, backward correlation and the prox epilogue are
//     the CUDA-core code of tnrd_stage.cuh.
#pragma once
#include "tnrd_stage.cuh"

namespace tnrd {
namespace tc {

constexpr int kG = 16;           // filters per MMA batch (MMA N)
constexpr int kS = 4;            // filters per RBF/backward sub-group
constexpr int kPW = 32;          // phi-region width (4 classes x 8 points)
constexpr int kPH = 32;          // phi-region height (2 bands of 16 rows)
constexpr int kBlocks = 8;       // 2 bands x 4 classes, M = 128 each
constexpr int kSPW = 36;         // sPhi row stride (floats)
constexpr int kNT = 256;         // 8 warps = 2 warpgroups
constexpr int kNSPLIT = 2;       // backward filter split (2 filters each)
constexpr int kTmemCols = 256;   // 2 buffers x 8 blocks x 16 columns

// instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, M=128, N=16
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kG >> 3) << 17) |
                            ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SWIZZLE_NONE, K-major shared-memory matrix descriptor (sm_100 version 1)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* v) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}

// Host-prepared forward GEMM operand per stage (tnrd_model_create): for
// batch b, tap row a, K-step kk (b = 8kk .. 8kk+7), precision p (0 hi, 1 lo):
// K-major [kc (2)][n (16)][4] = kf_n[a][8kk + 4kc + e] (zero for b >= m),
// kf = rot180(k) the correlation form of the true convolution.
template <int MS>
struct TcCfg {
    static constexpr int R = MS / 2;
    static constexpr int KSTEPS = (MS + 7) / 8;           // K = 8 per MMA
    static constexpr int TH = (MS == 9) ? 24 : (MS == 7 ? 26 : (MS == 5 ? 28 : 30));
    static constexpr int TW = (MS == 9) ? 24 : (MS == 7 ? 26 : 28);
    static constexpr int RB = 2;
    static constexpr int OBX = (TW + 3) / 4;
    static constexpr int OBY = (TH + RB - 1) / RB;
    static constexpr int ITEMS = OBX * OBY * kNSPLIT;
    static_assert(ITEMS <= kNT, "backward items must fit the CTA");
    static_assert(TH + 2 * R <= kPH && TW + 2 * R <= kPW, "tile + halo must fit the phi region");
    static_assert(4 * OBX + 2 * R <= kSPW && RB * OBY + 2 * R <= kPH, "backward reads outside sPhi");
    static constexpr int UR = kPH + 2 * R;                // u rows
    static constexpr int CW = 32 + 8 * KSTEPS - 4;        // class-copy width (floats)
    static constexpr int CS = round_up(CW, 4);            // class-copy row stride
    static constexpr int COPY = UR * CS;                  // floats per class copy
    static constexpr int BOP = 2 * kG * 4;                // floats per (a, kk, prec) operand
    static constexpr int BBATCH = MS * KSTEPS * 2 * BOP;  // floats per batch
    static constexpr int KP = round_up(MS * MS, 4);
    static constexpr int SPHI = kPH * kSPW;
    // shared layout (floats)
    static constexpr int OFF_COPY = 0;                    // [4 classes][2 prec][COPY]
    static constexpr int OFF_B = OFF_COPY + 8 * COPY;     // [2 buf][BBATCH]
    static constexpr int OFF_TAP = OFF_B + 2 * BBATCH;    // [2 buf][kS][KP]
    static constexpr int OFF_PHI = OFF_TAP + 2 * kS * KP; // [kS][SPHI]
    static constexpr int OFF_TAB = OFF_PHI + kS * SPHI;   // [kS][tab_stride]
    static size_t smem_bytes(int tab_stride) {
        return sizeof(float) * (size_t)(OFF_TAB + kS * tab_stride) + 64;  // + barriers
    }
};

template <int MS>
__global__ void __launch_bounds__(kNT, 2) stage_kernel_tc(const StageArgs p, const float* __restrict__ bop) {
    using C = TcCfg<MS>;
    constexpr int R = C::R;
    extern __shared__ __align__(128) float smem[];
    float* sCopy = smem + C::OFF_COPY;
    float* sB = smem + C::OFF_B;
    float* sTap = smem + C::OFF_TAP;
    float* sPhi = smem + C::OFF_PHI;
    float* sTab = smem + C::OFF_TAB;
    const int tabsz = kS * p.tab_stride;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTab + tabsz);  // [2] batch MMAs done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int img = blockIdx.z;
    const int Y0 = blockIdx.y * C::TH;
    const int X0 = blockIdx.x * C::TW;
    const float* __restrict__ uin = p.u_in + (int64_t)img * p.img_stride;
    const float* __restrict__ fin = p.f + (int64_t)img * p.img_stride;
    float* __restrict__ uout = p.u_out + (int64_t)img * p.img_stride;
    const bool top_halo = p.flags & 0x2u;
    const bool bot_halo = p.flags & 0x4u;
    const int nbatch = p.ngroups;                 // batches of kG filters
    const int nsub = (p.nk + kS - 1) / kS;        // real sub-groups of kS filters

    auto prefetch_b = [&](int b, int buf) {       // forward GEMM operand of batch b
        const float* gb = bop + (size_t)b * C::BBATCH;
        float* sb = sB + buf * C::BBATCH;
        for (int i = tid; i < C::BBATCH / 4; i += kNT) cp_async16(sb + 4 * i, gb + 4 * i);
    };
    auto prefetch_sub = [&](int sg, int buf) {    // taps + RBF tables of sub-group sg
        const float* gt = p.taps + (size_t)sg * kS * C::KP;
        float* st = sTap + buf * kS * C::KP;
        for (int i = tid; i < kS * C::KP / 4; i += kNT) cp_async16(st + 4 * i, gt + 4 * i);
        const float* gb = p.tab + (size_t)sg * tabsz;   // single buffer: used only by the RBF phase
        for (int i = tid; i < tabsz / 4; i += kNT) cp_async16(sTab + 4 * i, gb + 4 * i);
    };

    // ---- setup: barriers, TMEM, operands ------------------------------------
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    prefetch_b(0, 0);
    if (nbatch > 1) prefetch_b(1, 1);
    prefetch_sub(0, 0);
    cp_async_commit();

    // A operand: u region (2r halo), staged in sPhi (free until the first
    // RBF phase), then class copies copy[o][prec][ur][j] = hi/lo(u_reg[ur][j + o])
    constexpr int UW = C::CW + 3;
    float* sU = sPhi;
    static_assert(C::UR * UW <= kS * C::SPHI, "u staging must fit sPhi");
    {
        const bool floor_in = p.flags & 0x1u;
        for (int i = tid; i < C::UR * UW; i += kNT) {
            const int uy = i / UW, ux = i - uy * UW;
            int Y = Y0 - 2 * R + uy;
            const int X = mirror_clamp(X0 - 2 * R + ux, p.W);
            if (Y < 0) Y = top_halo ? max(Y, -2 * R) : mirror_clamp(Y, p.H);
            else if (Y >= p.H) Y = bot_halo ? min(Y, p.H - 1 + 2 * R) : mirror_clamp(Y, p.H);
            float v = __ldg(uin + (int64_t)Y * p.ld + X);
            if (floor_in) v = fmaxf(v, p.u0_floor);
            sU[i] = v;
        }
    }
    __syncthreads();
    for (int i = tid; i < 4 * C::COPY; i += kNT) {
        const int o = i / C::COPY;
        const int rem = i - o * C::COPY;
        const int ur = rem / C::CS, j = rem - ur * C::CS;
        const float u = (j < C::CW) ? sU[ur * UW + j + o] : 0.0f;
        const float hi = tf32_rna(u);
        sCopy[(o * 2 + 0) * C::COPY + rem] = hi;
        sCopy[(o * 2 + 1) * C::COPY + rem] = tf32_rna(u - hi);  // |u - hi - lo| <= 2^-22 |u|
    }
    cp_async_wait_all();
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    // one elected thread issues batch b: 2 bands x m taps x K-steps x 3
    // passes x 4 classes (classes innermost: consecutive MMAs hit different
    // accumulators)
    auto issue_batch = [&](int b) {
        const int buf = b & 1;
        const float* sb = sB + buf * C::BBATCH;
        for (int band = 0; band < 2; ++band) {
            for (int a = 0; a < MS; ++a) {
                for (int kk = 0; kk < C::KSTEPS; ++kk) {
                    const uint32_t arow = (uint32_t)((16 * band + a) * C::CS + 8 * kk) * 4u;
                    const float* bb = sb + ((a * C::KSTEPS + kk) * 2) * C::BOP;
                    const uint64_t bhi = make_desc(smem_u32(bb), kG * 16, 128);
                    const uint64_t blo = make_desc(smem_u32(bb + C::BOP), kG * 16, 128);
#pragma unroll
                    for (int pass = 0; pass < 3; ++pass) {
#pragma unroll
                        for (int o = 0; o < 4; ++o) {
                            const int prec = pass == 1 ? 1 : 0;
                            const uint64_t ad = make_desc(smem_u32(sCopy + (o * 2 + prec) * C::COPY) + arow,
                                                          16, C::CS * 4);
                            const uint32_t d = tmem + (uint32_t)(buf * 128 + (band * 4 + o) * kG);
                            const uint32_t acc = (a | kk | pass) ? 1u : 0u;
                            mma_tf32(d, ad, pass == 2 ? blo : bhi, acc);
                        }
                    }
                }
            }
        }
        mma_commit(&bars[buf]);
    };
    if (tid == 0) issue_batch(0);

    // tile touches a mirrored image edge? (phi halo fix-up needed)
    const bool fix_l = X0 - R < 0;
    const bool fix_r = X0 + C::TW + R > p.W;
    const bool fix_t = !top_halo && (Y0 - R < 0);
    const bool fix_b = !bot_halo && (Y0 + C::TH + R > p.H);
    const bool need_fix = fix_l || fix_r || fix_t || fix_b;

    // backward item of this thread
    const bool has_item = tid < C::ITEMS;
    const int obx = tid % C::OBX, oby = (tid / C::OBX) % C::OBY, split = tid / (C::OBX * C::OBY);
    const int ox0 = obx * 4, oy0 = oby * C::RB;
    float force[C::RB][4];
#pragma unroll
    for (int r = 0; r < C::RB; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) force[r][c] = 0.0f;

    const int wg = warp >> 2, q = warp & 3;
    for (int sg = 0; sg < nsub; ++sg) {
        const int b = sg / (kG / kS), s = sg % (kG / kS), sbuf = sg & 1;
        if (s == 0) {
            mbar_wait(&bars[b & 1], (b >> 1) & 1);   // batch b in TMEM
            fence_after();
            if (b + 2 < nbatch) prefetch_b(b + 2, b & 1);  // its B buffer is free now
            cp_async_commit();
            if (tid == 0 && b + 1 < nbatch) issue_batch(b + 1);
        }
        // ---- RBF: TMEM -> phi -> sPhi (4 filters) ----------------------------
        const float* tabg = sTab;
#pragma unroll 1
        for (int blk = wg; blk < kBlocks; blk += 2) {
            float z[kS];
            tmem_ld4(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)((b & 1) * 128 + blk * kG + s * kS), z);
            const int row = 32 * q + lane;
            const int py = 16 * (blk >> 2) + (row >> 3);
            const int px = 4 * (row & 7) + (blk & 3);
#pragma unroll
            for (int j = 0; j < kS; ++j)
                sPhi[j * C::SPHI + py * kSPW + px] = rbf_poly(z[j], tabg + j * p.tab_stride, p);
        }
        fence_before();
        __syncthreads();  // sPhi complete; tables of sg and taps of sg-1 free
        if (sg + 1 < nsub) prefetch_sub(sg + 1, sbuf ^ 1);   // lands during the bwd
        cp_async_commit();
        // ---- phi halo outside the image = mirror of in-image phi -------------
        if (need_fix) {
            // only the out-of-image band of the phi region is rewritten: rows
            // [0, nt) and [h0, kPH) and, for the rows in between, columns
            // [0, nl) and [w0, kPW); sources are in-image (mirror).
            const int nt_ = fix_t ? min(R, kPH) : 0;
            const int h0 = fix_b ? max(nt_, min(kPH, p.H - (Y0 - R))) : kPH;
            const int nl_ = fix_l ? R : 0;
            const int w0 = fix_r ? max(nl_, min(kPW, p.W - (X0 - R))) : kPW;
            const int full_rows = nt_ + (kPH - h0);
            const int mid_rows = h0 - nt_;
            const int per_f = full_rows * kPW + mid_rows * (nl_ + kPW - w0);
            for (int i = tid; i < kS * per_f; i += kNT) {
                const int j = i / per_f;
                int rem = i - j * per_f;
                int py, px;
                if (rem < full_rows * kPW) {
                    const int rr = rem / kPW;
                    px = rem - rr * kPW;
                    py = rr < nt_ ? rr : h0 + (rr - nt_);
                } else {
                    rem -= full_rows * kPW;
                    const int wcols = nl_ + kPW - w0;
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
                    sPhi[j * C::SPHI + py * kSPW + px] = sPhi[j * C::SPHI + spy * kSPW + spx];
                }
            }
            __syncthreads();
        }
        // ---- backward: force += corr(phi_j, k_j), 2 filters per item ---------
        if (has_item) {
            const float* tapg = sTap + sbuf * kS * C::KP;
#pragma unroll 1
            for (int jj = 0; jj < kS / kNSPLIT; ++jj) {
                const int j = split * (kS / kNSPLIT) + jj;
                if (sg * kS + j >= p.nk) break;
                float k[MS * MS];
                {
                    const float4* t4 = reinterpret_cast<const float4*>(tapg + j * C::KP);
#pragma unroll
                    for (int qq = 0; qq < C::KP / 4; ++qq) {
                        const float4 v = t4[qq];
                        if (4 * qq + 0 < MS * MS) k[4 * qq + 0] = v.x;
                        if (4 * qq + 1 < MS * MS) k[4 * qq + 1] = v.y;
                        if (4 * qq + 2 < MS * MS) k[4 * qq + 2] = v.z;
                        if (4 * qq + 3 < MS * MS) k[4 * qq + 3] = v.w;
                    }
                }
                constexpr int NV = (4 + 2 * R + 3) / 4;
                const float* ph = sPhi + j * C::SPHI;
#pragma unroll
                for (int rr = 0; rr < C::RB + 2 * R; ++rr) {
                    float v[4 * NV];
                    const float* src = ph + (oy0 + rr) * kSPW + ox0;
#pragma unroll
                    for (int qq = 0; qq < NV; ++qq) {
                        const float4 t = lds128(src + 4 * qq);
                        v[4 * qq] = t.x; v[4 * qq + 1] = t.y; v[4 * qq + 2] = t.z; v[4 * qq + 3] = t.w;
                    }
#pragma unroll
                    for (int a = 0; a < MS; ++a) {
                        const int ro = rr - a;
                        if (ro >= 0 && ro < C::RB) {
#pragma unroll
                            for (int bb = 0; bb < MS; ++bb) {
                                const float kk = k[a * MS + bb];
#pragma unroll
                                for (int c = 0; c < 4; ++c) force[ro][c] = fmaf(kk, v[c + bb], force[ro][c]);
                            }
                        }
                    }
                }
            }
        }
        cp_async_wait_all();
        fence_async_smem();
        __syncthreads();  // bwd done with sPhi/taps; next tables/taps/B landed
    }

    // ---- release TMEM (all batches were waited on) ------------------------------
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
    }

    // ---- reduce the filter splits, epilogue ------------------------------------
    float* red = sPhi;
    const int slot = (oby * C::OBX + obx) * C::RB * 4;
    if (has_item && split > 0) {
#pragma unroll
        for (int r = 0; r < C::RB; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                red[(split - 1) * C::OBX * C::OBY * C::RB * 4 + slot + r * 4 + c] = force[r][c];
    }
    __syncthreads();
    if (!has_item || split > 0) return;
    for (int s2 = 1; s2 < kNSPLIT; ++s2)
#pragma unroll
        for (int r = 0; r < C::RB; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                force[r][c] += red[(s2 - 1) * C::OBX * C::OBY * C::RB * 4 + slot + r * 4 + c];

    const bool out_force = p.flags & 0x8u;
    const bool check_f = p.flags & 0x10u;
    bool bad = false;
    uint32_t fbits = 0;
#pragma unroll
    for (int r = 0; r < C::RB; ++r) {
        const int oy = oy0 + r, Y = Y0 + oy;
        if (oy >= C::TH || Y >= p.H) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int ox = ox0 + c, X = X0 + ox;
            if (ox >= C::TW || X >= p.W) continue;
            float res;
            if (out_force) {
                res = force[r][c];
            } else {
                float u = __ldg(uin + (int64_t)Y * p.ld + X);  // exact u (the copies are split)
                if (p.flags & 0x1u) u = fmaxf(u, p.u0_floor);
                const float fv = __ldg(fin + (int64_t)Y * p.ld + X);
                if (check_f) {
                    if (!isfinite(fv)) fbits |= 0x1u;
                    else if (fv < 0.0f) fbits |= 0x2u;
                }
                res = reaction(u, force[r][c], fv, p);
            }
            if (!isfinite(res)) bad = true;
            uout[(int64_t)Y * p.ld + X] = res;
        }
    }
    if (bad) atomicMin(p.status, (uint32_t)p.stage);
    if (fbits) atomicAnd(p.status + 1, ~fbits);
}

}  // namespace tc
}  // namespace tnrd

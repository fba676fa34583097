// tnrd_stage_zf.cuh -- "z-field" stage: the forward filter bank on the
// tensor cores over the whole image, then a CUDA-core RBF + adjoint + prox
// kernel fed by TMA.  Same operator as tnrd_stage.cuh (reference
// diffusion.py:184-194):
//
//   z_i   = conv2d(u, k_i)                      imageops.py:53-72
//   phi_i = sum_j w_ij exp(-(z_i-mu_j)^2/2g^2)  influence.py:40-45
//   force = sum_i conv2d(phi_i, rot180(k_i))    diffusion.py:178-180 (phi
//           mirror padded itself)
//   u'    = prox_idiv(u - force, f, lam)        speckle.py:111-121
//
// Why two kernels: the fused CUDA-core kernel executes ~5,800 FFMA per
// pixel-stage (78% of its instructions, profiles/r02_zf), i.e. it sits on
// the direct method's FMA floor; the forward half of that is a GEMM.  Doing
// it per output tile on the tensor cores (tnrd_stage_tc*.cuh) recomputes z
// on every tile's phi halo and ties the TMEM accumulators to the tile, which
// held those kernels to small tiles and 2 CTAs/SM.  Here:
//
//   zfield_kernel (tcgen05): z_i at every image point exactly once, all
//       nk_pad filters in one N = nk_pad MMA, 3-piece tf32 split of u and k
//       with the 6 leading cross terms (error below fp32 rounding), fp32
//       accumulation in TMEM; epilogue tcgen05.ld -> float4 stores of the
//       z planes [img][filter][R + y][x] (L2-resident for one 512^2 image).
//   zstage_kernel (CUDA cores): per output tile and filter group, one TMA
//       3-D box load of the group's z planes over the tile + r halo (double
//       buffered, mbarrier complete_tx), phi = RBF(z) in place, mirror the
//       out-of-image phi band, adjoint correlation into register-resident
//       force, prox epilogue.  No u staging and no forward FMAs.
//
// The A operand needs no im2col: for point class o = x mod 4 the A rows of
// the 8 class-o points of an image row are overlapping 32-byte windows of a
// class-shifted copy of the u row (K-major SWIZZLE_NONE core matrices with
// rows 16 B apart: LBO = 16 B, SBO = copy row stride), one M = 128 MMA per
// (class, tap row, K-step, pass) covering 16 rows x 8 points.
#pragma once
#include <cuda.h>
#include "tnrd_stage.cuh"
#include "tnrd_stage_tc.cuh"

namespace tnrd {
namespace zf {

using tc::fence_after;
using tc::fence_async_smem;
using tc::fence_before;
using tc::make_desc;
using tc::mbar_init;
using tc::mma_commit;
using tc::smem_u32;
using tc::tf32_rna;

constexpr int kBandRows = 16;   // z rows per zfield CTA (MMA M = 16 rows x 8 points)
constexpr int kBandCols = 32;   // z columns per zfield CTA (4 classes x 8 points)
constexpr int kZThreads = 128;  // 4 warps = the 4 TMEM lane quadrants
constexpr int kPieces = 3;      // tf32 pieces of u and of k
constexpr int kMaxPass = 6;

// pass table: pass p multiplies u piece (pass_u >> 2p & 3) by k piece
// (pass_k >> 2p & 3)
struct ZArgs {
    const float* u_in;
    int64_t ld, img_stride;
    int H, W;
    uint32_t flags;        // 0x1 floor the input, 0x2 / 0x4 top / bottom halo rows exist
    float u0_floor;
    const float* bop;      // [m][ks][kPieces][2 kc][np][4]
    float* z;              // [img][np][H + 2r][zld]: z(y, x) at row y + r, column x + r
    int64_t zld, zplane, zimg;
    int zrow0;             // z rows computed: image rows [zrow0, zrow0 + gridDim.y * 16) clipped to zrow_end
    int zrow_end;
    int npass;
    uint32_t pass_u, pass_k;
};

template <int MS, int NP>
struct ZCfg {
    static constexpr int R = MS / 2;
    static constexpr int KS = (MS + 7) / 8;                 // K = 8 per MMA
    static constexpr int UR = kBandRows + 2 * R;            // u rows per band
    static constexpr int CW = kBandCols + 8 * KS - 4;       // class-copy width (floats)
    static constexpr int CS = round_up(CW, 4);              // class-copy row stride
    static constexpr int UW = CW + 3;                       // staged u width
    static constexpr int COPY = UR * CS;                    // floats per (class, piece)
    static constexpr int BOP = 2 * NP * 4;                  // floats per (a, kk, piece)
    static constexpr int BSZ = MS * KS * kPieces * BOP;     // B operand floats
    static constexpr int TMEM_COLS = 4 * NP <= 64 ? 64 : (4 * NP <= 128 ? 128 : (4 * NP <= 256 ? 256 : 512));
    // shared layout (floats): B | copies[4][kPieces] | u stage | barrier
    static constexpr int OFF_B = 0;
    static constexpr int OFF_COPY = BSZ;
    static constexpr int OFF_U = OFF_COPY + 4 * kPieces * COPY;
    static constexpr int OFF_BAR = round_up(OFF_U + UR * UW, 4);
    static constexpr size_t smem_bytes() { return sizeof(float) * (size_t)OFF_BAR + 32; }
    // instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, M = 128, N = NP
    static constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) |
                                       ((uint32_t)(128 >> 4) << 24);
    static_assert(NP % 16 == 0 && NP <= 128, "MMA N");
};

__device__ __forceinline__ void mma_tf32_id(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// bounded wait: a lost arrive traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
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

// ---- zfield_kernel: z_i = conv2d(u, k_i) on tensor cores -------------------
template <int MS, int NP>
__global__ void __launch_bounds__(kZThreads) zfield_kernel(const ZArgs p) {
    using C = ZCfg<MS, NP>;
    constexpr int R = C::R;
    extern __shared__ __align__(128) float smem[];
    float* sB = smem + C::OFF_B;
    float* sCopy = smem + C::OFF_COPY;
    float* sU = smem + C::OFF_U;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int img = blockIdx.z;
    // bands start r columns left of a multiple of 32: z of image column x
    // lives at plane column x + r, so this band's float4 stores are aligned
    // and so are the zstage TMA boxes (their x start must be a multiple of 4)
    const int X0 = blockIdx.x * kBandCols - R;
    const int Y0 = p.zrow0 + blockIdx.y * kBandRows;   // first z row of the band (may be < 0)
    const float* __restrict__ uin = p.u_in + (int64_t)img * p.img_stride;

    // parameters do not depend on the previous stage: load before the PDL wait
    for (int i = tid; i < C::BSZ / 4; i += kZThreads) cp_async16(sB + 4 * i, p.bop + 4 * i);
    cp_async_commit();
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    pdl_wait();     // the previous stage wrote u_in; the previous zstage read z
    pdl_trigger();

    // u rows [Y0 - R, Y0 + 16 + R), columns [X0 - R, X0 - R + UW): mirrored at
    // image edges, real halo rows of a strip, floored on the first stage
    const bool top_halo = p.flags & 0x2u, bot_halo = p.flags & 0x4u, floor_in = p.flags & 0x1u;
    for (int i = tid; i < C::UR * C::UW; i += kZThreads) {
        const int uy = i / C::UW, ux = i - uy * C::UW;
        int Y = Y0 - R + uy;
        const int X = mirror_clamp(X0 - R + ux, p.W);
        if (Y < 0) Y = top_halo ? max(Y, -2 * R) : mirror_clamp(Y, p.H);
        else if (Y >= p.H) Y = bot_halo ? min(Y, p.H - 1 + 2 * R) : mirror_clamp(Y, p.H);
        float v = __ldg(uin + (int64_t)Y * p.ld + X);
        sU[i] = floor_in ? fmaxf(v, p.u0_floor) : v;
    }
    __syncthreads();
    // class copies, split into 3 tf32 pieces: copy[o][piece][ur][j] = piece(u[ur][j + o])
    for (int i = tid; i < 4 * C::COPY; i += kZThreads) {
        const int o = i / C::COPY;
        const int rem = i - o * C::COPY;
        const int ur = rem / C::CS, j = rem - ur * C::CS;
        const float v = (j < C::CW) ? sU[ur * C::UW + j + o] : 0.0f;
        const float h0 = tf32_rna(v);
        const float r1 = v - h0;
        const float h1 = tf32_rna(r1);
        const float h2 = tf32_rna(r1 - h1);
        float* dst = sCopy + (o * kPieces) * C::COPY + rem;
        dst[0] = h0;
        dst[C::COPY] = h1;
        dst[2 * C::COPY] = h2;
    }
    cp_async_wait_all();
    fence_async_smem();   // generic-proxy smem writes -> visible to the tensor core
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (tid == 0) {
        for (int o = 0; o < 4; ++o) {
            const uint32_t d = tmem + (uint32_t)(o * NP);
            for (int a = 0; a < MS; ++a)
                for (int kk = 0; kk < C::KS; ++kk)
                    for (int ps = 0; ps < p.npass; ++ps) {
                        const int pu = (p.pass_u >> (2 * ps)) & 3, pk = (p.pass_k >> (2 * ps)) & 3;
                        const uint64_t ad = make_desc(smem_u32(sCopy + (o * kPieces + pu) * C::COPY +
                                                               a * C::CS + 8 * kk),
                                                      16, C::CS * 4);
                        const uint64_t bd = make_desc(smem_u32(sB + ((a * C::KS + kk) * kPieces + pk) * C::BOP),
                                                      NP * 16, 128);
                        mma_tf32_id(d, ad, bd, C::kIdesc, (a | kk | ps) ? 1u : 0u);
                    }
        }
        mma_commit(bar);
    }
    mbar_wait_bounded(bar, 0);
    fence_after();

    // epilogue: lane l of warp w = M row 32w + l = band row 4w + l/8, point
    // k = l % 8 of every class -> z at x = X0 + 4k .. +3 as one float4
    const int zr = Y0 + 4 * warp + (lane >> 3);       // image row of this thread's points
    const int zc = X0 + R + 4 * (lane & 7);           // plane column of its first point
    const bool store = zr < p.zrow_end && zc < p.zld;
    float* zrow = p.z + (int64_t)img * p.zimg + (int64_t)(zr + R) * p.zld + zc;
    const uint32_t tbase = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll 1
    for (int c = 0; c < NP / 16; ++c) {
        uint32_t v[4][16];
#pragma unroll
        for (int o = 0; o < 4; ++o) tmem_ld16(tbase + (uint32_t)(o * NP + 16 * c), v[o]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (store) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                __stcg(reinterpret_cast<float4*>(zrow + (int64_t)(16 * c + j) * p.zplane),
                       make_float4(__uint_as_float(v[0][j]), __uint_as_float(v[1][j]),
                                   __uint_as_float(v[2][j]), __uint_as_float(v[3][j])));
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(C::TMEM_COLS));
    }
}

// ---- zstage_kernel: phi = RBF(z), adjoint correlation, prox ----------------

template <int MS, int TH, int TW, int RB, int NT, int F>
struct ZSCfg {
    static constexpr int R = MS / 2;
    static constexpr int PH = TH + 2 * R;              // phi rows
    static constexpr int PW = round_up(TW + 2 * R, 4); // phi cols (TMA box width, 16 B multiple)
    static constexpr int SPHI = PH * PW;
    static constexpr int KK = MS * MS;
    static constexpr int KP = round_up(KK, 4);
    static constexpr int NV = (4 + 2 * R + 3) / 4;
    static constexpr int OBX = TW / 4;
    static constexpr int OBY = TH / RB;
    static constexpr int NSPLIT = NT / (OBX * OBY);
    static_assert(OBX * OBY * NSPLIT == NT && F % NSPLIT == 0, "output blocks x filter split must cover the CTA");
    static_assert(PW <= 256 && PH <= 256, "TMA box");
    // the backward's float4 row reads stay inside the phi region
    static_assert(TW - 4 + 4 * NV <= PW, "backward reads");
    // z / phi buffer stride: the TMA destination must be 128-byte aligned
    static constexpr int ZBUF = round_up(F * SPHI, 32);
    // shared (floats): zphi[2][ZBUF] | taps[2][F*KP] | tab[2][F*tab_stride] | bars
    static size_t smem_bytes(int tab_stride) {
        return sizeof(float) * (size_t)(2 * ZBUF + 2 * F * KP + 2 * F * tab_stride) + 64;
    }
};

struct ZStageArgs {
    StageArgs s;
    int np;          // z planes per image
};

__device__ __forceinline__ void tma_load_3d(float* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

template <int MS, int TH, int TW, int RB, int NT, int F, int MINB>
__global__ void __launch_bounds__(NT, MINB) zstage_kernel(const ZStageArgs za,
                                                          const __grid_constant__ CUtensorMap zmap) {
    using C = ZSCfg<MS, TH, TW, RB, NT, F>;
    using SC = StageCfg<MS, TH, TW, 1, RB, NT, F>;   // same phi geometry for fix-up / backward
    static_assert(SC::PH == C::PH && SC::PW == C::PW, "phi geometry");
    constexpr int R = C::R;
    const StageArgs& p = za.s;
    extern __shared__ __align__(128) float smem[];
    float* sZ = smem;                                  // [2][ZBUF]
    float* sTap = sZ + 2 * C::ZBUF;
    float* sTab = sTap + 2 * F * C::KP;
    const int tabsz = F * p.tab_stride;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sTab + 2 * tabsz);

    const int tid = threadIdx.x;
    const int img = blockIdx.z;
    const int Y0 = blockIdx.y * TH;
    const int X0 = blockIdx.x * TW;
    const bool top_halo = p.flags & 0x2u;
    const bool bot_halo = p.flags & 0x4u;
    const int ng = p.ngroups;
    constexpr uint32_t kBoxBytes = (uint32_t)(F * C::SPHI * sizeof(float));

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&zmap)) : "memory");
    }
    prefetch_group<SC, F, NT>(p, sTap, sTab, 0, 0, tid);
    __syncthreads();
    pdl_wait();     // z of this stage (zfield) and u_in are complete
    pdl_trigger();
    // z planes of group g: box (PW, PH, F) over image rows / columns from
    // (Y0 - R, X0 - R), i.e. plane coordinates (X0, Y0) (multiple of 4 in x,
    // which TMA requires of the innermost start coordinate)
    auto issue = [&](int g, int buf) {
        fence_async_smem();
        mbar_expect_tx(&bars[buf], kBoxBytes);
        tma_load_3d(sZ + buf * C::ZBUF, &zmap, X0, Y0, img * za.np + g * F, &bars[buf]);
    };
    if (tid == 0) {
        issue(0, 0);
        if (ng > 1) issue(1, 1);
    }

    const int split = tid / (C::OBX * C::OBY);
    const int obx = tid % C::OBX, oby = (tid / C::OBX) % C::OBY;
    const int ox0 = obx * 4, oy0 = oby * RB;
    float force[RB][4];
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) force[r][c] = 0.0f;

    for (int g = 0; g < ng; ++g) {
        const int buf = g & 1;
        cp_async_wait_all();
        __syncthreads();  // tables of g landed; group g-1 is done with its z buffer and tables
        if (tid == 0 && g >= 1 && g + 1 < ng) issue(g + 1, buf ^ 1);
        if (g + 1 < ng) prefetch_group<SC, F, NT>(p, sTap, sTab, g + 1, buf ^ 1, tid);
        const float* tapg = sTap + buf * F * C::KP;
        const float* tabg = sTab + buf * tabsz;
        float* ph = sZ + buf * C::ZBUF;
        mbar_wait_bounded(&bars[buf], (g >> 1) & 1);
        // phi = RBF(z) in place, 4 points per item
        constexpr int Q = C::SPHI / 4;
        for (int i = tid; i < F * Q; i += NT) {
            const int fi = i / Q;
            const uint32_t tb = rbf_table_base(tabg + fi * p.tab_stride, p);
            float4 z = *reinterpret_cast<const float4*>(ph + 4 * i);
            z.x = rbf_poly_s(z.x, tb, p);
            z.y = rbf_poly_s(z.y, tb, p);
            z.z = rbf_poly_s(z.z, tb, p);
            z.w = rbf_poly_s(z.w, tb, p);
            *reinterpret_cast<float4*>(ph + 4 * i) = z;
        }
        __syncthreads();
        fix_phi<SC, F, NT, TH, TW>(p, ph, Y0, X0, top_halo, bot_halo, tid);
        backward_group<SC, MS, RB, F>(ph, tapg, split, ox0, oy0, force);
    }
    if (!reduce_splits<SC, RB>(sZ, split, obx, oby, force)) return;

    const float* __restrict__ uin = p.u_in + (int64_t)img * p.img_stride;
    const float* __restrict__ fin = p.f + (int64_t)img * p.img_stride;
    float* __restrict__ uout = p.u_out + (int64_t)img * p.img_stride;
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
            const int64_t off = (int64_t)Y * p.ld + X;
            float u = __ldg(uin + off);
            if (p.flags & 0x1u) u = fmaxf(u, p.u0_floor);
            finish_pixel(p, u, force[r][c], fin, uout, off, bad, fbits);
        }
    }
    report(p, bad, fbits);
}

}  // namespace zf
}  // namespace tnrd

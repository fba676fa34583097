// tnrd_stage_adj.cuh -- diffusion stage with the ADJOINT filter bank on the
// tensor cores (tcgen05, sm_100a): two kernels per stage, opt-in mode 12.
// Same operator as tnrd_stage.cuh (reference diffusion.py:184-194):
//
//   z_i   = conv2d(u, k_i)                      imageops.py:53-72
//   phi_i = sum_j w_ij exp(-(z_i-mu_j)^2/2g^2)  influence.py:40-45
//   force = sum_i conv2d(phi_i, rot180(k_i))    diffusion.py:178-180 (phi
//           mirror padded itself)
//   u'    = prox_idiv(u - force, f, lam)        speckle.py:111-121
//
// Why: the fused CUDA-core kernel is FMA-pipe bound, and a build without its
// backward runs 1.5x faster, so the adjoint -- the
// accuracy-safe half -- is worth moving off the FMA pipe.
// It is a GEMM: psi(p, tap) = sum_i phi_i(p) k_i[tap] (M = pixels, K = Nk,
// N = m^2 taps), followed by a shifted sum force(q) = sum_tap psi(q + tap -
// r, tap).  The fused kernel cannot host it (TMEM / shared memory, DESIGN.md
// 4.8), so the stage is split at phi:
//
//   phi_kernel   (CUDA cores)  z and phi = RBF(z) for every image pixel
//       exactly once (no halo recompute: a CTA computes its 64 x 64 tile
//       only), with the parameter-space taps, FFMA2 filter pairs and the
//       cubic RBF table of stage_kernel_pt; phi is written to global memory
//       in the GEMM's A-operand layout -- per region row and 4-filter chunk,
//       one float4 (4 filters) per pixel: Phi[img][y + r][kc][x + r][4] --
//       including the mirrored copies outside the image (the reference pads
//       phi itself), so the adjoint kernel has no edge cases.
//   adj_kernel   (tcgen05)     a CTA owns a 4-strip column group (4 x (32 -
//       2r) output columns) over a range of rows and walks the region rows:
//       a TMA warp streams the row's phi (K-major core matrices, 32 pixels
//       per strip with a 2r overlap between strips) into a 3-slot ring; the
//       four epilogue warps split it into tf32 hi + lo; an MMA warp issues
//       the 3xTF32 GEMM D[128 pixels x taps] += hi Khi + lo Khi + hi Klo
//       (kind::tf32, fp32 accumulation in TMEM, two accumulators); the
//       epilogue warps read D with tcgen05.ld (lane = pixel), sum the taps of
//       a filter row across lanes with a 6-step shuffle chain, accumulate the
//       m filter rows in a register window that slides down the image, and
//       finish each completed output row (u - force, reaction, status
//       flags, store).
//
// All sums run in a fixed order (the MMA's own reduction is deterministic),
// so results are bit-reproducible; they differ from the CUDA-core kernels by
// the 3xTF32 products (~2^-21 relative) and the summation order.
#pragma once
#include "tnrd_stage.cuh"

namespace tnrd {
namespace adj {

constexpr int kStrips = 4;        // strips per adjoint CTA = TMEM lane quadrants = epilogue warps
constexpr int kStripW = 32;       // pixels per strip (one warp)
constexpr int kSlots = 4;         // raw phi row ring (TMA destination, pixel-major)
constexpr int kOpSlots = 2;       // A-operand buffers (tf32 hi and lo of a row, K-major core matrices)
constexpr int kAdjThreads = 320;  // 4 epilogue warps + TMA warp + MMA warp + 4 converter warps
constexpr int kPhiTile = 64;      // phi_kernel tile (square)
constexpr int kPhiThreads = 256;

struct AdjArgs {
    float* phi;            // [img][H + 2r][kc][xp][4]
    int64_t phi_row;       // floats per region row   (kc * xp * 4)
    int64_t phi_img;       // floats per image
    int xp;                // padded pixels per region row
    int kc;                // 4-filter chunks (nk_pad / 4)
    const float* bop;      // [ks][2 prec][2 kc][NB][4] tf32 hi / lo of k_i[tap]
    int rows_per_cta;      // output rows per adjoint CTA
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// SWIZZLE_NONE, K-major shared-memory matrix descriptor (sm_100 version 1):
// core matrix = 8 rows x 16 B, contiguous; lbo = bytes between core matrices
// adjacent in K, sbo = bytes between core matrices adjacent in M / N
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// bounded wait: a lost arrive traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- phi_kernel -------------------------------------------------------------

// forward configuration without a halo: the phi region IS the tile (the
// members forward_group_pt / forward_block_fp / stage_u_tile read)
template <int MS, int RF>
struct PhiCfg {
    static constexpr int R = MS / 2;
    static constexpr int PH = kPhiTile;
    static constexpr int PW = kPhiTile;
    static constexpr int UR = PH + 2 * R;
    static constexpr int US = padded_stride(PW + round_up(2 * R, 4), RF, PW / 4);
    static constexpr int NV = (4 + 2 * R + 3) / 4;
    static constexpr int KK = MS * MS;
    static constexpr int KP = round_up(KK, 4);
    static constexpr int NBX = PW / 4;
    static constexpr int NBY = PH / RF;
    static constexpr int NBLK = NBX * NBY;
    static constexpr int SU = UR * US;
    static constexpr int SPHI = PH * PW;
    static_assert(PH % RF == 0, "forward blocks must tile the region");
    // shared layout (floats): u | phi[4] | tab3[2]
    static size_t smem_bytes(int tab3_stride) {
        return sizeof(float) * ((size_t)SU + 4 * (size_t)SPHI + 2 * (size_t)tab3_stride);
    }
};

// one 64 x 64 tile: phi of all filters, 4 at a time, to the global Phi array
template <int MS, int RF, int TM, class TB>
__global__ void __launch_bounds__(kPhiThreads, 2) phi_kernel(const StageArgs p, const AdjArgs q,
                                                            const __grid_constant__ TB tk) {
    using C = PhiCfg<MS, RF>;
    constexpr int R = C::R;
    constexpr int NT = kPhiThreads;
    extern __shared__ __align__(16) float smem[];
    float* sU = smem;
    float* sPhi = sU + C::SU;
    float* sTab = sPhi + 4 * C::SPHI;
    const int tabsz = 2 * p.tab3_stride;
    const int tid = threadIdx.x;
    const int img = blockIdx.z;
    const int Y0 = blockIdx.y * kPhiTile, X0 = blockIdx.x * kPhiTile;
    const float* __restrict__ uin = p.u_in + (int64_t)img * p.img_stride;
    const float* kp = tk.k;
    constexpr int GS = TapLayout<MS, C::KP, 2, TM>::group;

    __shared__ __align__(8) uint64_t tbar;
    if (tid == 0) {
        tbar_init(&tbar);
        tbar_fetch(sTab, p.tab3, tabsz, &tbar);
    }
    __syncthreads();
    // (Y0 + R, X0 + R): stage_u_tile's origin is 2R above / left of its argument
    stage_u_tile<C, NT>(p, sU, uin, Y0 + R, X0 + R, false, false, tid);

    // mirrored copies (the reference pads phi itself): an in-image pixel
    // within r of an image edge also fills its reflections outside the image
    const bool edge = Y0 < R || X0 < R || Y0 + kPhiTile + R > p.H || X0 + kPhiTile + R > p.W;
    float* phig = q.phi + (int64_t)img * q.phi_img;
    const int ngroups = p.ngroups;   // pairs of filters
    for (int g = 0; g < ngroups; ++g) {
        tbar_wait(&tbar, g & 1);
        __syncthreads();   // table g landed; the flush of the previous chunk is done with sPhi
        forward_group_pt<C, MS, RF, 2, NT, true, TM>(p, sU, sPhi + (g & 1) * 2 * C::SPHI, kp + g * GS, sTab, tid);
        __syncthreads();
        if (tid == 0 && g + 1 < ngroups) tbar_fetch(sTab, p.tab3 + (size_t)(g + 1) * tabsz, tabsz, &tbar);
        if (!(g & 1) && g + 1 < ngroups) continue;   // second pair of the chunk still to come
        const int kc = g >> 1;
        const bool half = !(g & 1);                  // odd pair count: the last chunk's upper half is zero
        for (int i = tid; i < C::SPHI; i += NT) {
            const int y = i / kPhiTile, x = i - y * kPhiTile;
            const int Y = Y0 + y, X = X0 + x;
            if (Y >= p.H || X >= p.W) continue;
            float4 v;
            v.x = sPhi[i];
            v.y = sPhi[C::SPHI + i];
            v.z = half ? 0.0f : sPhi[2 * C::SPHI + i];
            v.w = half ? 0.0f : sPhi[3 * C::SPHI + i];
            // chunk-major rows [y + r][kc][x + r][4]: a warp's 32 pixels are one
            // 512 B store (a pixel-major layout, one bulk copy per row for the
            // consumer, made this kernel 2.8x slower: 16 B stores at a 192 B stride)
            float* row = phig + (int64_t)kc * q.xp * 4;
            const int64_t pxs = 4;
            if (!edge) {
                *reinterpret_cast<float4*>(row + (int64_t)(Y + R) * q.phi_row + (int64_t)(X + R) * pxs) = v;
            } else {
                // rows {Y, top mirror, bottom mirror} x columns {X, left, right mirror}
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int ya = a == 0 ? Y : (a == 1 ? -1 - Y : 2 * p.H - 1 - Y);
                    if ((a == 1 && Y >= R) || (a == 2 && Y < p.H - R)) continue;
#pragma unroll
                    for (int b = 0; b < 3; ++b) {
                        const int xb = b == 0 ? X : (b == 1 ? -1 - X : 2 * p.W - 1 - X);
                        if ((b == 1 && X >= R) || (b == 2 && X < p.W - R)) continue;
                        *reinterpret_cast<float4*>(row + (int64_t)(ya + R) * q.phi_row + (int64_t)(xb + R) * pxs) = v;
                    }
                }
            }
        }
    }
}

// ---- adj_kernel -------------------------------------------------------------

template <int MS>
struct AdjCfg {
    static constexpr int R = MS / 2;
    static constexpr int TAPS = MS * MS;
    static constexpr int NB = round_up(TAPS, 16);             // MMA N
    static constexpr int PITCH = kStripW - 2 * R;              // output columns per strip
    static constexpr int GW = kStrips * PITCH;                 // output columns per CTA
    static constexpr int TMEM_COLS = 2 * NB <= 32 ? 32 : (2 * NB <= 64 ? 64 : (2 * NB <= 128 ? 128 : 256));
    static constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NB >> 3) << 17) |
                                       ((uint32_t)(128 >> 4) << 24);
    static constexpr int NPX = GW + 2 * R;                     // region pixels per row of the group
    static constexpr int KCS = 128 * 16 + 16;                  // bytes between 4-filter chunks of an A
                                                               // operand (padded: the converters'
                                                               // chunk-strided stores spread over the banks)
    // shared layout (bytes): B | raw [kSlots] | A hi [kOpSlots] | A lo [kOpSlots] | barriers | tmem slot
    __host__ __device__ static constexpr size_t b_bytes(int kc) { return (size_t)(kc / 2) * 2 * 2 * NB * 16; }
    __host__ __device__ static constexpr size_t raw_bytes(int kc) { return (size_t)NPX * kc * 16; }
    __host__ __device__ static constexpr size_t op_bytes(int kc) { return (size_t)kc * KCS; }
    static size_t smem_bytes(int kc) {
        return b_bytes(kc) + kSlots * raw_bytes(kc) + 2 * kOpSlots * op_bytes(kc) + 256;
    }
};

template <int MS>
__global__ void __launch_bounds__(kAdjThreads, 1) adj_kernel(const StageArgs p, const AdjArgs q) {
    using C = AdjCfg<MS>;
    constexpr int R = C::R;
    constexpr int NB = C::NB;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int KC = q.kc, KS = q.kc / 2;
    const uint32_t rawbytes = (uint32_t)C::raw_bytes(KC), opbytes = (uint32_t)C::op_bytes(KC);
    float* sB = reinterpret_cast<float*>(smem_raw);
    unsigned char* sRaw = smem_raw + C::b_bytes(KC);
    unsigned char* sHi = sRaw + (size_t)kSlots * rawbytes;
    unsigned char* sLo = sHi + (size_t)kOpSlots * opbytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sLo + (size_t)kOpSlots * opbytes);
    uint64_t* full = bars;                        // [kSlots] TMA landed
    uint64_t* rawfree = bars + kSlots;            // [kSlots] converters done with the raw row
    uint64_t* conv = bars + 2 * kSlots;           // [2] hi / lo of a row written
    uint64_t* convfree = conv + kOpSlots;         // [2] the MMAs that read the operand buffer are done
    uint64_t* accfull = convfree + kOpSlots;      // [2] accumulator complete
    uint64_t* accfree = accfull + 2;              // [2] accumulator read by the epilogue
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfree + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int img = blockIdx.z;
    const int o0 = blockIdx.y * q.rows_per_cta;                 // first output row
    const int o1 = min(p.H, o0 + q.rows_per_cta);
    const int nrows = o1 - o0 + 2 * R;                          // region rows o0 .. o1 - 1 + 2R
    const int c0 = blockIdx.x * C::GW;                          // first region column of the group

    if (tid == 0) {
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&rawfree[i], kStrips);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&conv[i], kStrips);
            mbar_init(&convfree[i], 1);
            mbar_init(&accfull[i], 1);
            mbar_init(&accfree[i], kStrips);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    // B operand (this stage's taps, tf32 hi / lo)
    {
        const int n4 = (int)(C::b_bytes(KC) / 16);
        const float4* src = reinterpret_cast<const float4*>(q.bop);
        float4* dst = reinterpret_cast<float4*>(sB);
        for (int i = tid; i < n4; i += kAdjThreads) dst[i] = __ldg(src + i);
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const float* phig = q.phi + (int64_t)img * q.phi_img;

    if (warp == 4) {
        // ---- TMA producer: region row o0 + j, columns c0 .. c0 + NPX - 1 of
        // every 4-filter chunk (KC contiguous pieces of NPX x 16 B) into slot
        // j % kSlots as raw[kc][px]
        if (lane == 0) {
            for (int j = 0; j < nrows; ++j) {
                const int slot = j % kSlots;
                if (j >= kSlots) mbar_wait(&rawfree[slot], ((j / kSlots) - 1) & 1);
                mbar_expect_tx(&full[slot], rawbytes);
                const float* src = phig + (int64_t)(o0 + j) * q.phi_row + (int64_t)c0 * 4;
                unsigned char* dst = sRaw + (size_t)slot * rawbytes;
                for (int kc = 0; kc < KC; ++kc)
                    bulk_g2s(dst + (size_t)kc * C::NPX * 16, src + (int64_t)kc * q.xp * 4, C::NPX * 16, &full[slot]);
            }
        }
    } else if (warp == 5) {
        // ---- MMA issuer: D[acc] = hi Khi + lo Khi + hi Klo over all K-steps
        if (lane == 0) {
            for (int j = 0; j < nrows; ++j) {
                const int b = j & 1;
                mbar_wait(&conv[b], (j >> 1) & 1);
                if (j >= 2) mbar_wait(&accfree[b], ((j >> 1) - 1) & 1);
                fence_after();
                const uint32_t d = tmem + (uint32_t)(b * NB);
                const uint32_t ahi = smem_u32(sHi + (size_t)b * opbytes);
                const uint32_t alo = smem_u32(sLo + (size_t)b * opbytes);
                for (int ks = 0; ks < KS; ++ks) {
                    const uint64_t dah = make_desc(ahi + (uint32_t)ks * 2 * C::KCS, C::KCS, 128);
                    const uint64_t dal = make_desc(alo + (uint32_t)ks * 2 * C::KCS, C::KCS, 128);
                    const uint32_t bb = smem_u32(sB) + (uint32_t)ks * (2 * 2 * NB * 16);
                    const uint64_t dbh = make_desc(bb, NB * 16, 128);
                    const uint64_t dbl = make_desc(bb + 2 * NB * 16, NB * 16, 128);
                    mma_tf32(d, dah, dbh, C::kIdesc, ks ? 1u : 0u);
                    mma_tf32(d, dal, dbh, C::kIdesc, 1u);
                    mma_tf32(d, dah, dbl, C::kIdesc, 1u);
                }
                mma_commit(&convfree[b]);
                mma_commit(&accfull[b]);
            }
        }
    } else if (warp >= 6) {
        // ---- converter warps: thread = region pixel px of the row; its KC
        // float4 (4 filters each) go, split into tf32 hi and lo = phi - hi, to
        // lane l1 of the K-major operand (strip s1 = px / PITCH, clamped) and,
        // in the 2R columns two strips share, also to lane l2 of the strip
        // on the left
        const int px = tid - 6 * 32;
        const int s1 = min(px / C::PITCH, kStrips - 1), r1 = px - C::PITCH * s1;
        const int l1 = kStripW * s1 + r1;
        const int l2 = (r1 < 2 * R && s1 >= 1) ? kStripW * (s1 - 1) + r1 + C::PITCH : -1;
        for (int j = 0; j < nrows; ++j) {
            const int slot = j % kSlots, b = j & 1;
            mbar_wait(&full[slot], (j / kSlots) & 1);
            if (j >= 2) mbar_wait(&convfree[b], ((j >> 1) - 1) & 1);   // row j - 2 multiplied
            if (px < C::NPX) {
                const float4* raw = reinterpret_cast<const float4*>(sRaw + (size_t)slot * rawbytes) + px;
                unsigned char* hi = sHi + (size_t)b * opbytes;
                unsigned char* lo = sLo + (size_t)b * opbytes;
                for (int kc = 0; kc < KC; ++kc) {
                    const float4 v = raw[kc * C::NPX];
                    float4 h, l;
                    h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
                    l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
                    const size_t o1b = (size_t)kc * C::KCS + (size_t)l1 * 16;
                    *reinterpret_cast<float4*>(hi + o1b) = h;
                    *reinterpret_cast<float4*>(lo + o1b) = l;
                    if (l2 >= 0) {
                        const size_t o2b = (size_t)kc * C::KCS + (size_t)l2 * 16;
                        *reinterpret_cast<float4*>(hi + o2b) = h;
                        *reinterpret_cast<float4*>(lo + o2b) = l;
                    }
                }
            }
            fence_async_smem();   // generic-proxy writes -> visible to the tensor core
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&conv[b]);
                mbar_arrive(&rawfree[slot]);
            }
        }
    } else {
        // ---- epilogue warps: warp w = strip w = TMEM lanes 32w..
        // output column of this lane and the rows' shared state
        const int X = c0 + warp * C::PITCH + lane;             // image column of lane's OUTPUT
        const bool col_ok = lane < C::PITCH && X < p.W;
        const float* __restrict__ uin = p.u_in + (int64_t)img * p.img_stride;
        const float* __restrict__ fin = p.f + (int64_t)img * p.img_stride;
        float* __restrict__ uout = p.u_out + (int64_t)img * p.img_stride;
        float* fout = p.force_out ? p.force_out + (int64_t)img * p.img_stride : nullptr;
        bool bad = false;
        uint32_t fbits = 0;
        float win[MS];    // output-row window: win[(j - a) mod MS] collects row o0 + j - a
#pragma unroll
        for (int i = 0; i < MS; ++i) win[i] = 0.0f;
        const uint32_t tlane = tmem + ((uint32_t)(32 * warp) << 16);

        for (int j0 = 0; j0 < nrows; j0 += MS) {
#pragma unroll
            for (int jj = 0; jj < MS; ++jj) {
                const int j = j0 + jj;
                if (j < nrows) {                      // warp-uniform
                    // u and f of the output row this step completes, loaded
                    // before the waits so their latency hides under them
                    const int Y = o0 + j - 2 * R;
                    const bool emit = j >= 2 * R && col_ok;
                    float u = 0.0f, fv = 0.0f;
                    if (emit) {
                        u = __ldg(uin + (int64_t)Y * p.ld + X);
                        fv = __ldg(fin + (int64_t)Y * p.ld + X);
                    }
                    const int acc = j & 1;
                    mbar_wait(&accfull[acc], (j >> 1) & 1);
                    fence_after();
                    float v[NB];
#pragma unroll
                    for (int c = 0; c < NB / 16; ++c) tmem_ld16(tlane + (uint32_t)(acc * NB + 16 * c), v + 16 * c);
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&accfree[acc]);
                    // filter row a: sum over b of psi(x + b, (a, b)) by a shuffle chain
#pragma unroll
                    for (int a = 0; a < MS; ++a) {
                        float t = v[a * MS + MS - 1];
#pragma unroll
                        for (int b = MS - 2; b >= 0; --b)
                            t = __shfl_down_sync(0xffffffffu, t, 1) + v[a * MS + b];
                        const int s = (jj - a + MS) % MS;
                        win[s] = a == 0 ? t : win[s] + t;
                    }
                    // output row o0 + j - 2R is complete
                    if (emit) {
                        if (p.flags & 0x1u) u = fmaxf(u, p.u0_floor);
                        finish_pixel_f(p, u, win[(jj + 1) % MS], fv, uout, (int64_t)Y * p.ld + X, bad, fbits, fout);
                    }
                }
            }
        }
        report(p, bad, fbits);
    }
    fence_before();
    __syncthreads();
    if (warp == 5) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(C::TMEM_COLS));
    }
}

}  // namespace adj
}  // namespace tnrd

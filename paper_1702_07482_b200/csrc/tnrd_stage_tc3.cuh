// tnrd_stage_tc3.cuh -- warp-specialised tcgen05 stage (forward GEMM on the
// tensor cores, RBF + backward on the CUDA cores) without CTA-wide barriers
// in the filter loop.
//
// Why: the phase-locked tcgen05 kernel (tnrd_stage_tc.cuh) issues 20% fewer
// instructions than the CUDA-core kernel but stalls on __syncthreads (22% of
// samples, 51% issue).  Here one CTA per SM runs
//   * 1 MMA warp: issues the 3xTF32 forward GEMM of 16-filter batches into a
//     double-buffered TMEM accumulator (2 x 256 columns = all of TMEM) and
//     streams the next batch's B operand with cp.async;
//   * 2 "halves" of 8 warps, ping-ponging over 4-filter sub-groups (half h
//     takes sub-groups h, h+2, ...): tcgen05.ld z -> RBF -> phi (own shared
//     slot) -> border mirror -> backward correlation into a per-half force
//     accumulator.  A half only synchronises with itself (named barrier
//     1 + h) and with the MMA warp through mbarriers (tmem_full: commit;
//     tmem_empty: one arrive per half), so one half computes while the other
//     waits.
// Geometry: phi region 32 x 64 (2 bands x 2 column groups x 4 classes = 16
// M=128 blocks), output tile (32 - 2r) x (64 - 2r) -> 26 x 58 for m = 7
// (phi points per output 1.36 instead of 1.51).
#pragma once
#include "tnrd_stage_tc.cuh"

namespace tnrd {
namespace tc3 {

using tc::fence_after;
using tc::fence_async_smem;
using tc::fence_before;
using tc::kIdesc;
using tc::make_desc;
using tc::mbar_init;
using tc::mma_commit;
using tc::mma_tf32;
using tc::smem_u32;
using tc::tf32_rna;
using tc::tmem_ld4;

constexpr int kG = 16;          // filters per MMA batch (N)
constexpr int kS = 4;           // filters per sub-group
constexpr int kPH = 32, kPW = 64;
constexpr int kBlocks = 16;     // 2 bands x 2 column groups x 4 classes
constexpr int kHalfWarps = 8;
constexpr int kNT = 32 * (2 * kHalfWarps + 1);  // 544: two halves + MMA warp
constexpr int kMmaWarp = 2 * kHalfWarps;
constexpr int kTmemCols = 512;  // 2 buffers x 16 blocks x 16 columns
constexpr int kSPW = 68;        // phi row stride

// bounded mbarrier wait: a protocol bug traps (~2 s) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
    const long long t0 = clock64();
    for (;;) {
        uint32_t done;
        // the suspend-time hint parks the warp in hardware until the phase
        // flips (or ~0.5 ms pass) instead of spinning on issue slots
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(500000u)
            : "memory");
        if (done) return;
        if (clock64() - t0 > 4000000000LL) __trap();
    }
}

__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync 0;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void half_sync(int h) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + h), "r"(32 * kHalfWarps) : "memory");
}

template <int MS>
struct Cfg {
    static constexpr int R = MS / 2;
    static constexpr int KSTEPS = (MS + 7) / 8;
    static constexpr int TH = kPH - 2 * R;
    static constexpr int TW = ((kPW - 2 * R) / 2) * 2;     // even
    static constexpr int RB = 2;
    static constexpr int OBX = (TW + 3) / 4;
    static constexpr int OBY = (TH + RB - 1) / RB;
    static constexpr int ITEMS = OBX * OBY;                // per half, all 4 filters
    static_assert(ITEMS <= 32 * kHalfWarps, "backward items must fit a half");
    static_assert(4 * OBX + 2 * R <= kSPW && RB * OBY + 2 * R <= kPH, "backward reads outside phi");
    static constexpr int UR = kPH + 2 * R;
    static constexpr int CW = kPW + 8 * KSTEPS - 4;        // class-copy width
    static constexpr int CS = round_up(CW, 4);
    static constexpr int COPY = UR * CS;
    static constexpr int BOP = 2 * kG * 4;
    static constexpr int BBATCH = MS * KSTEPS * 2 * BOP;
    static constexpr int KP = round_up(MS * MS, 4);
    static constexpr int SPHI = kPH * kSPW;
    static constexpr int OFF_COPY = 0;                          // [4][2][COPY]
    static constexpr int OFF_B = OFF_COPY + 8 * COPY;           // [2][BBATCH]
    static constexpr int OFF_TAP = OFF_B + 2 * BBATCH;          // [2 halves][kS][KP]
    static constexpr int OFF_PHI = OFF_TAP + 2 * kS * KP;       // [2 halves][kS][SPHI]
    static constexpr int OFF_TAB = OFF_PHI + 2 * kS * SPHI;     // [2 halves][kS][tab_stride]
    static size_t smem_bytes(int tab_stride) {
        return sizeof(float) * (size_t)(OFF_TAB + 2 * kS * tab_stride) + 128;
    }
};

template <int MS>
__global__ void __launch_bounds__(kNT, 1) stage_kernel_tc3(const StageArgs p, const float* __restrict__ bop) {
    using C = Cfg<MS>;
    constexpr int R = C::R;
    extern __shared__ __align__(128) float smem[];
    float* sCopy = smem + C::OFF_COPY;
    float* sB = smem + C::OFF_B;
    const int tabsz = kS * p.tab_stride;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_TAB + 2 * tabsz);
    uint64_t* tmem_full = bars;       // [2] MMA commit
    uint64_t* tmem_empty = bars + 2;  // [2] one arrive per half
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

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
    const int nbatch = p.ngroups;
    const int nsub = (p.nk + kS - 1) / kS;

    // ---- setup (all warps) ------------------------------------------------------
    if (tid == 0) {
        mbar_init(&tmem_full[0], 1);
        mbar_init(&tmem_full[1], 1);
        mbar_init(&tmem_empty[0], 2);
        mbar_init(&tmem_empty[1], 2);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    // u region staged in the phi slots (free until the first RBF phase), then
    // split class copies copy[o][prec][ur][j] = hi/lo(u_reg[ur][j + o])
    constexpr int UW = C::CW + 3;
    float* sU = smem + C::OFF_PHI;
    static_assert(C::UR * UW <= 2 * kS * C::SPHI, "u staging must fit the phi slots");
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
        sCopy[(o * 2 + 1) * C::COPY + rem] = tf32_rna(u - hi);
    }
    fence_async_smem();
    fence_before();
    __syncthreads();  // copies ready, sU dead, barriers initialised, TMEM allocated
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == kMmaWarp) {
        // ================= MMA warp =====================================================
        auto load_b = [&](int b) {
            const float* gb = bop + (size_t)b * C::BBATCH;
            float* sb = sB + (b & 1) * C::BBATCH;
            for (int i = lane; i < C::BBATCH / 4; i += 32) cp_async16(sb + 4 * i, gb + 4 * i);
            cp_async_commit();
            cp_async_wait_all();
            fence_async_smem();
            __syncwarp();
        };
        load_b(0);
        if (nbatch > 1) load_b(1);
        for (int b = 0; b < nbatch; ++b) {
            const int buf = b & 1;
            if (b >= 2) mbar_wait_bounded(&tmem_empty[buf], ((b >> 1) - 1) & 1);
            fence_after();
            if (lane == 0) {
                const float* sb = sB + buf * C::BBATCH;
                for (int band = 0; band < 2; ++band)
                    for (int a = 0; a < MS; ++a)
                        for (int kk = 0; kk < C::KSTEPS; ++kk) {
                            const float* bb = sb + ((a * C::KSTEPS + kk) * 2) * C::BOP;
                            const uint64_t bhi = make_desc(smem_u32(bb), kG * 16, 128);
                            const uint64_t blo = make_desc(smem_u32(bb + C::BOP), kG * 16, 128);
                            for (int pass = 0; pass < 3; ++pass)
                                for (int cg = 0; cg < 2; ++cg)
#pragma unroll
                                    for (int o = 0; o < 4; ++o) {
                                        const int prec = pass == 1 ? 1 : 0;
                                        const uint32_t arow =
                                            (uint32_t)((16 * band + a) * C::CS + 32 * cg + 8 * kk) * 4u;
                                        const uint64_t ad = make_desc(
                                            smem_u32(sCopy + (o * 2 + prec) * C::COPY) + arow, 16, C::CS * 4);
                                        const int blk = (band * 2 + cg) * 4 + o;
                                        const uint32_t d = tmem + (uint32_t)(buf * 256 + blk * kG);
                                        mma_tf32(d, ad, pass == 2 ? blo : bhi, (a | kk | pass) ? 1u : 0u);
                                    }
                        }
                mma_commit(&tmem_full[buf]);
            }
            __syncwarp();
            // B of batch b+1 goes into the buffer batch b-1 used: wait for it
            if (b >= 1 && b + 1 < nbatch) {
                mbar_wait_bounded(&tmem_full[(b - 1) & 1], ((b - 1) >> 1) & 1);
                load_b(b + 1);
            }
        }
    } else {
        // ================= halves: RBF + backward ========================================
        const int h = warp / kHalfWarps;              // 0 or 1
        const int htid = tid - h * 32 * kHalfWarps;   // 0..255
        const int hw = warp - h * kHalfWarps;         // warp within the half
        const int wg = hw >> 2, q = hw & 3;           // TMEM lane quarter q
        float* sPhi = smem + C::OFF_PHI + h * kS * C::SPHI;
        float* sTab = smem + C::OFF_TAB + h * tabsz;
        float* sTap = smem + C::OFF_TAP + h * kS * C::KP;
        auto prefetch_sub = [&](int sg) {
            const float* gt = p.taps + (size_t)sg * kS * C::KP;
            for (int i = htid; i < kS * C::KP / 4; i += 32 * kHalfWarps) cp_async16(sTap + 4 * i, gt + 4 * i);
            const float* gb = p.tab + (size_t)sg * tabsz;
            for (int i = htid; i < tabsz / 4; i += 32 * kHalfWarps) cp_async16(sTab + 4 * i, gb + 4 * i);
            cp_async_commit();
        };

        const bool fix_l = X0 - R < 0;
        const bool fix_r = X0 + C::TW + R > p.W;
        const bool fix_t = !top_halo && (Y0 - R < 0);
        const bool fix_b = !bot_halo && (Y0 + C::TH + R > p.H);
        const bool need_fix = fix_l || fix_r || fix_t || fix_b;

        const bool has_item = htid < C::ITEMS;
        const int obx = htid % C::OBX, oby = htid / C::OBX;
        const int ox0 = obx * 4, oy0 = oby * C::RB;
        float force[C::RB][4];
#pragma unroll
        for (int r = 0; r < C::RB; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) force[r][c] = 0.0f;

        if (h < nsub) prefetch_sub(h);
        for (int sg = h; sg < nsub; sg += 2) {
            const int b = sg / (kG / kS), s = sg % (kG / kS), buf = b & 1;
            cp_async_wait_all();
            half_sync(h);                                  // taps/tables of sg landed for the half
            mbar_wait_bounded(&tmem_full[buf], (b >> 1) & 1);
            fence_after();
            // ---- RBF: TMEM -> phi (this half's slot), 2 blocks (8 z) per pass ---
            {
                const int row = 32 * q + lane;
                const uint32_t tbase = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * 256 + s * kS);
                const int prow = (row >> 3) * kSPW + 4 * (row & 7);   // phi offset within a block
#pragma unroll 1
                for (int blk = wg * 8; blk < wg * 8 + 8; blk += 2) {
                    float z[2][kS];
                    tmem_ld4(tbase + (uint32_t)(blk * kG), z[0]);
                    tmem_ld4(tbase + (uint32_t)((blk + 1) * kG), z[1]);
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        const int b2 = blk + h2;
                        const int off = 16 * (b2 >> 3) * kSPW + 32 * ((b2 >> 2) & 1) + (b2 & 3) + prow;
#pragma unroll
                        for (int j = 0; j < kS; ++j)
                            sPhi[j * C::SPHI + off] = rbf_poly(z[h2][j], sTab + j * p.tab_stride, p);
                    }
                }
            }
            fence_before();
            half_sync(h);                                  // slot complete; TMEM reads of sg done
            // this half's last sub-group of batch b releases the TMEM buffer
            const bool last_of_batch = (s + 2 >= kG / kS) || (sg + 2 >= nsub);
            if (last_of_batch && htid == 0) mbar_arrive(&tmem_empty[buf]);
            // ---- phi halo outside the image = mirror of in-image phi -----------
            if (need_fix) {
                const int nt_ = fix_t ? R : 0;
                const int h0 = fix_b ? max(nt_, min(kPH, p.H - (Y0 - R))) : kPH;
                const int nl_ = fix_l ? R : 0;
                const int w0 = fix_r ? max(nl_, min(kPW, p.W - (X0 - R))) : kPW;
                const int full_rows = nt_ + (kPH - h0);
                const int mid_rows = h0 - nt_;
                const int per_f = full_rows * kPW + mid_rows * (nl_ + kPW - w0);
                for (int i = htid; i < kS * per_f; i += 32 * kHalfWarps) {
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
                half_sync(h);
            }
            // ---- backward over the 4 filters of the slot -------------------------
            if (has_item) {
#pragma unroll 1
                for (int j = 0; j < kS; ++j) {
                    if (sg * kS + j >= p.nk) break;
                    float k[MS * MS];
                    {
                        const float4* t4 = reinterpret_cast<const float4*>(sTap + j * C::KP);
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
            half_sync(h);                                  // slot, taps and tables free again
            if (sg + 2 < nsub) prefetch_sub(sg + 2);
        }
        // ---- combine the halves, epilogue (half 0) ---------------------------------
        float* red = smem + C::OFF_PHI;                    // both slots are free after the loop
        cta_sync();                            // (MMA warp joins below)
        const int slot = (oby * C::OBX + obx) * C::RB * 4;
        if (h == 1 && has_item) {
#pragma unroll
            for (int r = 0; r < C::RB; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) red[slot + r * 4 + c] = force[r][c];
        }
        cta_sync();
        if (h == 0 && has_item) {
#pragma unroll
            for (int r = 0; r < C::RB; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) force[r][c] += red[slot + r * 4 + c];
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
                        float u = __ldg(uin + (int64_t)Y * p.ld + X);
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
        cta_sync();
        return;
    }
    // MMA warp: join the three CTA barriers of the halves' epilogue, then free TMEM
    cta_sync();
    cta_sync();
    cta_sync();
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
}

}  // namespace tc3
}  // namespace tnrd

// tnrd_stage_fused.cuh -- all T stages of one despeckle in ONE persistent
// launch, scheduled as a dataflow over (stage, tile) for small grids.
//
// The per-stage split path (stage_kernel_split + stage_reduce_kernel) pays
// every stage's ramp and tail: stage t+1 starts only when the whole of
// stage t is reduced.  But a tile of stage t+1 needs only its 3 x 3 tile
// neighbourhood of stage t (the stage's receptive radius m - 1 is below the
// 64-pixel tile).  Here a persistent grid claims work from one global
// sequence of (stage, tile, filter-group pair) claims, ordered by
// tile + D * stage, so stage t+1's first tiles are claimed while stage t's
// last tiles are still running:
//
//   * a claim computes the partial forces of two filter groups of one tile
//     (the split kernel's unit body) and adds 2 to the tile's counter;
//   * the CTA that completes a tile's last group (counter == ngroups) sums
//     its ngroups partials IN GROUP ORDER (cp.async-staged, thread-private
//     ring) and runs the epilogue -- u_{t+1} of the tile -- then publishes
//     the tile's done flag (release);
//   * a claim of stage t > 0 first waits (acquire, bounded spin) for the
//     done flags of its tile's neighbourhood in stage t - 1.
//
// Claims are taken in sequence order by resident CTAs and depend only on
// earlier claims, so the waits always terminate.  The summation order is the
// split kernel's, so results are bit-identical to the per-stage split path.
// Counters and flags are cleared by the last CTA to exit.
#pragma once
#include "tnrd_stage.cuh"

namespace tnrd {
namespace fused {

struct FusedArgs {
    const StageArgs* st;   // [T] per-stage arguments (u_in, u_out, tables, flags)
    const int* seq;        // [nclaims] (t << 24) | (tile << 6) | g0
    int nclaims;
    int T;
    int claim_groups;      // filter groups per claim
    float* part0;          // partial forces of even stages: [tiles][ngroups][TH*TW]
    float* part1;          // ... of odd stages
    uint32_t* cnt;         // [T][tiles] groups done
    uint32_t* done;        // [T][tiles] tile reduced (0/1)
    uint32_t* ctl;         // [0] claim cursor, [1] CTAs exited
    int tiles_x, tiles_y, tiles;
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// bounded spin: a dependency that never arrives traps (reported as a CUDA
// error) instead of hanging the GPU
__device__ __forceinline__ void wait_flag(const uint32_t* p, uint32_t want) {
    const long long t0 = clock64();
    while (ld_acquire(p) < want) {
        __nanosleep(100);
        if (clock64() - t0 > (1ll << 33)) asm volatile("trap;");
    }
}

__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_n() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#ifdef TNRD_FUSED_TRACE
// per CTA: total, waiting, reducing, staging (clock64 cycles), claims
__device__ long long g_fused_trace[4096][5];
#endif

template <int MS, int TH, int TW, int RF, int RB, int NT, bool FAST, int F, int MINB>
__global__ void __launch_bounds__(NT, MINB) despeckle_fused_kernel(const FusedArgs fa) {
#ifdef TNRD_FUSED_TRACE
    const long long tr0 = clock64();
    long long trw = 0, trr = 0, trs = 0, trn = 0;
#endif
    using C = StageCfg<MS, TH, TW, RF, RB, NT, F>;
    constexpr int R = C::R;
    constexpr int TPX = TH * TW;
    constexpr int QPT = TPX / 4 / NT;     // pixel quads per thread in the reduction
    // partial groups in flight per thread: as many as sU + sPhi hold (3-4)
    constexpr int RING = (C::SU + F * C::SPHI) / (QPT * NT * 4) < 4 ? (C::SU + F * C::SPHI) / (QPT * NT * 4) : 4;
    static_assert(RING >= 2, "reduction ring needs two slots");
    static_assert(TPX % (4 * NT) == 0, "tile quads must split evenly over the CTA");
    static_assert(RING * QPT * NT * 4 <= C::SU + F * C::SPHI, "reduction ring must fit in sU + sPhi");
    extern __shared__ __align__(16) float smem[];
    float* sU = smem;
    float* sPhi = sU + C::SU;
    float* sTap = sPhi + F * C::SPHI;
    float* sTab = sTap + 2 * F * C::KP;
    __shared__ StageArgs sp;
    __shared__ int s_claim, s_last;
    const int tid = threadIdx.x;
    const int split = tid / (C::OBX * C::OBY);
    const int obx = tid % C::OBX, oby = (tid / C::OBX) % C::OBY;
    const int ox0 = obx * 4, oy0 = oby * RB;
    const int tpi = fa.tiles_x * fa.tiles_y;   // tiles per image

    // claims are taken one ahead: the atomic for claim k+1 is in flight while
    // claim k runs
    if (tid == 0) s_claim = (int)atomicAdd(fa.ctl, 1u);
    for (;;) {
        __syncthreads();   // s_claim visible; the previous claim is done with smem and sp
        const int c = s_claim;
        if (c >= fa.nclaims) break;
        uint32_t pend = 0u;
        if (tid == 0) pend = atomicAdd(fa.ctl, 1u);   // consumed at the end of this claim
        const int e = fa.seq[c];
        const int t = e >> 24, tile = (e >> 6) & 0x3FFFF, g0 = e & 0x3F;
        // this stage's arguments into shared memory
        {
            const int* src = reinterpret_cast<const int*>(fa.st + t);
            int* dst = reinterpret_cast<int*>(&sp);
            for (int i = tid; i < (int)(sizeof(StageArgs) / sizeof(int)); i += NT) dst[i] = src[i];
        }
        const int img = tile / tpi, trem = tile - img * tpi;
        const int ty = trem / fa.tiles_x, tx = trem - ty * fa.tiles_x;
        // stage t reads u_t = the output of stage t - 1 on the 3 x 3 tile
        // neighbourhood: lanes 0-8 of warp 0 wait for those tiles (acquire)
#ifdef TNRD_FUSED_TRACE
        const long long trw0 = clock64();
        ++trn;
#endif
        if (t > 0 && tid < 32) {
            const int dy = tid / 3 - 1, dx = tid % 3 - 1;
            const int yy = ty + dy, xx = tx + dx;
            if (tid < 9 && yy >= 0 && yy < fa.tiles_y && xx >= 0 && xx < fa.tiles_x)
                wait_flag(fa.done + (size_t)(t - 1) * fa.tiles + img * tpi + yy * fa.tiles_x + xx, 1u);
            __syncwarp();
        }
        __syncthreads();   // sp copied; dependencies satisfied
#ifdef TNRD_FUSED_TRACE
        trw += clock64() - trw0;
        const long long trs0 = clock64();
#endif
        const StageArgs& p = sp;
        const int ng = p.ngroups;
        const int g1 = min(g0 + fa.claim_groups, ng);
        const bool top_halo = p.flags & 0x2u;
        const bool bot_halo = p.flags & 0x4u;
        const int Y0 = ty * TH, X0 = tx * TW;
        prefetch_group<C, F, NT>(p, sTap, sTab, g0, 0, tid);
        stage_u_tile<C, NT, true>(p, sU, p.u_in + (int64_t)img * p.img_stride, Y0, X0, top_halo,
                                  bot_halo, tid);
        float* part = (t & 1) ? fa.part1 : fa.part0;
        int buf = 0;
#ifdef TNRD_FUSED_TRACE
        cp_async_wait_all();
        __syncthreads();
        trs += clock64() - trs0;
#endif
        for (int g = g0; g < g1; ++g) {
            cp_async_wait_all();
            __syncthreads();   // params + u tile in smem; previous group done with sPhi
            if (g + 1 < g1) prefetch_group<C, F, NT>(p, sTap, sTab, g + 1, buf ^ 1, tid);
            const float* tapg = sTap + buf * F * C::KP;
            const float* tabg = sTab + buf * F * p.tab_stride;
            forward_group<C, MS, RF, F, FAST>(p, sU, sPhi, tapg, tabg, tid);
            __syncthreads();
            fix_phi<C, F, NT, TH, TW>(p, sPhi, Y0, X0, top_halo, bot_halo, tid);
            float force[RB][4];
#pragma unroll
            for (int r = 0; r < RB; ++r)
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) force[r][cc] = 0.0f;
            backward_group<C, MS, RB, F>(sPhi, tapg, split, ox0, oy0, force);
            if (reduce_splits<C, RB>(sPhi, split, obx, oby, force)) {
                float* dst = part + ((size_t)tile * ng + g) * TPX + oy0 * TW + ox0;
#pragma unroll
                for (int r = 0; r < RB; ++r)
                    __stcg(reinterpret_cast<float4*>(dst + r * TW),
                           make_float4(force[r][0], force[r][1], force[r][2], force[r][3]));
            }
            buf ^= 1;
        }
        // publish the groups; the CTA completing the tile reduces it
        __threadfence();
        __syncthreads();   // also: everyone is done with sU / sPhi
        if (tid == 0) {
            const uint32_t before = atomicAdd(fa.cnt + (size_t)t * fa.tiles + tile, (uint32_t)(g1 - g0));
            s_last = before + (uint32_t)(g1 - g0) == (uint32_t)ng;
        }
        __syncthreads();
        if (tid == 0) s_claim = (int)pend;   // read after the loop-top barrier
        if (!s_last) continue;
#ifdef TNRD_FUSED_TRACE
        const long long trr0 = clock64();
#endif
        __threadfence();   // acquire side of the other CTAs' partial stores
        // ---- reduction of the tile: partials summed in group order --------
        float4* ring = reinterpret_cast<float4*>(sU);   // [RING][QPT][NT], thread-private slots
        const float* src = part + (size_t)tile * ng * TPX;
        auto issue = [&](int g) {
            if (g < ng) {
#pragma unroll
                for (int q = 0; q < QPT; ++q)
                    cp_async16_cg(ring + ((g % RING) * QPT + q) * NT + tid,
                                  src + (size_t)g * TPX + 4 * (tid + q * NT));
            }
            cp_async_commit();   // (empty groups keep the count uniform)
        };
#pragma unroll
        for (int g = 0; g < RING - 1; ++g) issue(g);
        float4 acc[QPT];
        for (int g = 0; g < ng; ++g) {
            issue(g + RING - 1);
            cp_async_wait_n<RING - 1>();   // group g has landed (own copies only)
#pragma unroll
            for (int q = 0; q < QPT; ++q) {
                const float4 v = ring[((g % RING) * QPT + q) * NT + tid];
                if (g == 0) {
                    acc[q] = v;
                } else {
                    acc[q].x += v.x; acc[q].y += v.y; acc[q].z += v.z; acc[q].w += v.w;
                }
            }
        }
        cp_async_wait_all();
        bool bad = false;
        uint32_t fbits = 0;
        const float* __restrict__ uin = p.u_in + (int64_t)img * p.img_stride;
        const float* __restrict__ fin = p.f + (int64_t)img * p.img_stride;
        float* __restrict__ uout = p.u_out + (int64_t)img * p.img_stride;
#pragma unroll
        for (int q = 0; q < QPT; ++q) {
            const int i = 4 * (tid + q * NT);
            const int oy = i / TW, ox = i - oy * TW;
            const int Y = Y0 + oy;
            if (Y >= p.H) continue;
            const float fa4[4] = {acc[q].x, acc[q].y, acc[q].z, acc[q].w};
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int X = X0 + ox + cc;
                if (X >= p.W) continue;
                const int64_t off = (int64_t)Y * p.ld + X;
                float u = __ldcg(uin + off);
                if (p.flags & 0x1u) u = fmaxf(u, p.u0_floor);
                finish_pixel(p, u, fa4[cc], fin, uout, off, bad, fbits);
            }
        }
        report(p, bad, fbits);
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicExch(fa.done + (size_t)t * fa.tiles + tile, 1u);
#ifdef TNRD_FUSED_TRACE
        trr += clock64() - trr0;
#endif
    }
#ifdef TNRD_FUSED_TRACE
    if (tid == 0 && blockIdx.x < 4096) {
        g_fused_trace[blockIdx.x][0] = clock64() - tr0;
        g_fused_trace[blockIdx.x][1] = trw;
        g_fused_trace[blockIdx.x][2] = trr;
        g_fused_trace[blockIdx.x][3] = trs;
        g_fused_trace[blockIdx.x][4] = trn;
    }
#endif
    // the last CTA out clears the cursor, counters and flags
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(fa.ctl + 1, 1u) == gridDim.x - 1) {
            for (int i = 0; i < fa.T * fa.tiles; ++i) {
                fa.cnt[i] = 0u;
                fa.done[i] = 0u;
            }
            fa.ctl[0] = 0u;
            __threadfence();
            fa.ctl[1] = 0u;
        }
    }
}

}  // namespace fused
}  // namespace tnrd

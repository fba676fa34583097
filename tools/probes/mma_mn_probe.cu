// Probe of tcgen05.mma kind::tf32 operand layouts (development tool, not
// part of the library): D[128x16] = A[128x8] (K-major, SWIZZLE_NONE) *
// B[8x16] with B either K-major or MN-major, optional K-row start shift.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// A: 128 x 8, A[m][k] = a_in[m*8+k]; stored K-major core matrices:
//   [kc(2)][mgroup(16)][8 rows][4]  -> LBO = 16*128 B, SBO = 128 B
// B (K x N = 8 x 16): b_in[k*16+n]
//   mode 0: K-major [kc(2)][ngroup(2)][8 rows n][4 k] -> LBO = 2*128, SBO = 128
//   mode 1: MN-major [ngroup(4)][krow(KR)][4 n], rows start at `shift`
//           -> LBO = 128 (8-row K groups contiguous), SBO = KR*16
__global__ void probe(const float* a_in, const float* b_in, float* d_out, int mode, int shift, uint32_t lbo, uint32_t sbo, int layout) {
    __shared__ __align__(128) float sA[128 * 8];
    __shared__ __align__(128) float sB[4 * 24 * 4];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    int tid = threadIdx.x;
    for (int i = tid; i < 128 * 8; i += 128) {
        int m = i / 8, k = i % 8, kc = k / 4, e = k % 4;
        sA[(kc * 16 + m / 8) * 32 + (m % 8) * 4 + e] = a_in[i];
    }
    for (int i = tid; i < 4 * 24 * 4; i += 128) sB[i] = 0.f;
    __syncthreads();
    const int KR = 24;
    for (int i = tid; i < 8 * 16; i += 128) {
        int k = i / 16, n = i % 16;
        if (mode == 0) sB[((k / 4) * 2 + n / 8) * 32 + (n % 8) * 4 + (k % 4)] = b_in[i];
        else if (layout == 0) sB[((n / 4) * KR + (k + shift)) * 4 + (n % 4)] = b_in[i];
        else if (layout == 1) sB[((k + shift) * 4 + n / 4) * 4 + (n % 4)] = b_in[i];      // [k][nchunk][4]
        else sB[(((k + shift) / 8) * 4 * 8 + (n / 4) * 8 + (k + shift) % 8) * 4 + (n % 4)] = b_in[i];  // [kgrp][nchunk][8 k][4 n]
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = slot;
    if (tid == 0) {
        uint64_t ad = mdesc(su32(sA), 16 * 128, 128);
        uint64_t bd;
        uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
        if (mode == 0) bd = mdesc(su32(sB), 2 * 128, 128);
        else { bd = mdesc(su32(sB) + shift * 16 * (layout == 1 ? 4 : 1), lbo, sbo); idesc |= (1u << 16); }
        asm volatile("{.reg .pred p; setp.ne.b32 p, 0, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[16];
    uint32_t taddr = tmem + ((uint32_t)((tid / 32) * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 16; ++n) d_out[tid * 16 + n] = __uint_as_float(r[n]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
    std::vector<float> a(128 * 8), b(8 * 16), d(128 * 16);
    for (int i = 0; i < 128 * 8; ++i) a[i] = (float)((i * 7) % 13 - 6);
    for (int i = 0; i < 8 * 16; ++i) b[i] = (float)((i * 5) % 11 - 5);
    float *da, *db, *dd;
    cudaMalloc(&da, a.size() * 4); cudaMalloc(&db, b.size() * 4); cudaMalloc(&dd, d.size() * 4);
    cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    struct Cfg { int mode, layout; uint32_t lbo, sbo; };
    std::vector<Cfg> cfgs = {{0, 0, 0, 0}};
    uint32_t vals[] = {16, 64, 128, 256, 384, 512, 1024};
    for (int layout = 0; layout < 3; ++layout)
        for (uint32_t l : vals)
            for (uint32_t s2 : vals) cfgs.push_back({1, layout, l, s2});
    for (auto c : cfgs)
        for (int shift = 0; shift < (c.mode ? 2 : 1); ++shift) {
            int mode = c.mode;
            cudaMemset(dd, 0, d.size() * 4);
            probe<<<1, 128>>>(da, db, dd, mode, shift, c.lbo, c.sbo, c.layout);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 16; ++n) {
                    double ref = 0;
                    for (int k = 0; k < 8; ++k) ref += a[m * 8 + k] * b[k * 16 + n];
                    maxerr = fmax(maxerr, fabs(ref - d[m * 16 + n]));
                }
            double dsum = 0; for (float v : d) dsum += fabs(v);
            if (maxerr == 0 || mode == 0 || dsum != 0)
                printf("sum|d|=%g ", dsum), printf("mode %d layout %d lbo %u sbo %u shift %d: %s max err %g\n", mode, c.layout, c.lbo, c.sbo,
                       shift, cudaGetErrorString(e), maxerr);
        }
    return 0;
}

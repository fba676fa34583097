// Throughput of tcgen05.mma kind::tf32 (cta_group::1, M = 128, K = 8, A and B
// K-major SWIZZLE_NONE in shared memory, D in TMEM) against N: the evidence
// for DESIGN.md 4.8's "a GEMM form of the 7x7 adjoint is smem-operand
// bound".  Every CTA (1 or 2 per SM) issues `iters` MMAs from one elected
// thread into one accumulator and commits once; prints MAC/clk/SM and the
// implied shared-memory operand bytes/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int N>
__global__ void __launch_bounds__(128) rate(int iters, unsigned long long* cycles) {
    __shared__ __align__(1024) float sA[128 * 8];
    __shared__ __align__(1024) float sB[N * 8];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 128 * 8; i += 128) sA[i] = 1e-3f * (i % 7);
    for (int i = tid; i < N * 8; i += 128) sB[i] = 1e-3f * (i % 5);
    constexpr int COLS = N < 32 ? 32 : N;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "n"(COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    unsigned long long t0 = clock64();
    if (tid == 0) {
        const uint64_t ad = mdesc(su32(sA), 16 * 128, 128);
        const uint64_t bd = mdesc(su32(sB), (N / 8) * 128, 128);
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        for (int i = 0; i < iters; ++i)
            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                         ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(i));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(su32(&bar)));
    unsigned long long t1 = clock64();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) atomicMax(cycles, t1 - t0);
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(COLS));
}

template <int N>
void run(int per_sm, int sms) {
    unsigned long long* dc;
    cudaMalloc(&dc, 8);
    const int iters = 4096;
    float best = 1e30f;
    unsigned long long cyc = 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int r = 0; r < 4; ++r) {
        cudaMemset(dc, 0, 8);
        cudaEventRecord(e0);
        rate<N><<<sms * per_sm, 128>>>(iters, dc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) { best = ms; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost); }
    }
    const double macs_cta = 128.0 * N * 8 * iters;
    const double per_clk_sm = macs_cta * per_sm / (double)cyc;
    const double bytes_mma = (128.0 * 8 + N * 8.0) * 4;
    printf("N=%3d CTAs/SM=%d: %7.1f MAC/clk/SM  (%5.1f clk per MMA per CTA), smem operand %6.1f B/clk/SM, "
           "%.1f TFLOP/s tf32 chip  [%s]\n", N, per_sm, per_clk_sm, (double)cyc / iters,
           bytes_mma * iters * per_sm / (double)cyc, 2.0 * macs_cta * sms * per_sm / (best * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(dc);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int per = 1; per <= 2; ++per) {
        run<16>(per, sms); run<32>(per, sms); run<64>(per, sms); run<128>(per, sms); run<256>(per, sms);
    }
    return 0;
}

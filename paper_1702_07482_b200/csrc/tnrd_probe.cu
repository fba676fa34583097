// tnrd_probe.cu -- on-box peak probes for the roofline denominators.
//
// MEASURED_PEAKS.json only carries HBM and bf16-GEMM peaks; the stage kernel
// is bound by the FP32 FMA and MUFU (ex2) pipes, so bench.py measures those
// two peaks with these saturating kernels (8 independent dependency chains
// per thread, 16 warps per SM) and reports the fraction against them.
#include <cuda_runtime.h>

#include <atomic>

#include "../../include/tnrd.h"

namespace {

__global__ void __launch_bounds__(256) probe_ffma(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], b, a);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 1234.5f) out[0] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) probe_ex2(float* out, int iters, float a) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-6f + j * 1e-3f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float y;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[j]));
            x[j] = y * a;  // FMUL keeps the value bounded; MUFU is the binding pipe
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 1234.5f) out[0] = s;
}

}  // namespace

extern "C" int tnrd_probe(int kind, int iters, int blocks_per_sm, void* stream, double* ops) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static float* sink = nullptr;
    if (!sink && cudaMalloc(&sink, sizeof(float)) != cudaSuccess) return TNRD_ECUDA;
    const int blocks = sms * (blocks_per_sm > 0 ? blocks_per_sm : 2);
    const double threads = (double)blocks * 256.0;
    if (kind == 0) {
        probe_ffma<<<blocks, 256, 0, (cudaStream_t)stream>>>(sink, iters, 0.999f, 1e-3f);
        if (ops) *ops = threads * iters * 16.0 * 2.0;  // FLOP (FMA = 2)
    } else {
        probe_ex2<<<blocks, 256, 0, (cudaStream_t)stream>>>(sink, iters, 0.5f);
        if (ops) *ops = threads * iters * 8.0;  // ex2 operations
    }
    return cudaGetLastError() == cudaSuccess ? TNRD_OK : TNRD_ECUDA;
}

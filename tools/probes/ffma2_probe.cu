// FFMA vs FFMA2 (fma.rn.f32x2, sm_100a) throughput probe: 8 independent
// chains per thread, 256 threads, 4 CTAs per SM.  Prints TFLOP/s (FMA = 2).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk(unsigned long long r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

// all-register operands (values from memory so nothing folds)
__global__ void __launch_bounds__(256) k_rrr(float* out, const float* in, int iters) {
    float x[8], y[8];
    for (int j = 0; j < 8; ++j) { x[j] = in[j]; y[j] = in[8 + j]; }
    float z = in[16];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], y[j], z);
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = fmaf(y[j], x[j], z);
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += x[j] + y[j];
    if (s == 1234.5f) out[0] = s;
}
// uniform operand (kernel parameter)
__global__ void __launch_bounds__(256) k_rur(float* out, const float* in, int iters, float a, float b) {
    float x[16];
    for (int j = 0; j < 16; ++j) x[j] = in[j];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, x[(j + 8) & 15]);
    }
    float s = 0; for (int j = 0; j < 16; ++j) s += x[j];
    if (s == 1234.5f) out[0] = s;
}
// FFMA2, uniform pair operand
__global__ void __launch_bounds__(256) k_ffma2_u(float* out, const float* in, int iters, float a, float b) {
    unsigned long long x[8];
    for (int j = 0; j < 8; ++j) x[j] = pk(in[2 * j], in[2 * j + 1]);
    const unsigned long long ab = pk(a, b);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma2(x[j], ab, x[(j + 4) & 7]);
    }
    float s = 0; for (int j = 0; j < 8; ++j) { float2 v = upk(x[j]); s += v.x + v.y; }
    if (s == 1234.5f) out[0] = s;
}
// FFMA2, register pair operand broadcast from one scalar register
__global__ void __launch_bounds__(256) k_ffma2_bc(float* out, const float* in, int iters) {
    unsigned long long x[8];
    for (int j = 0; j < 8; ++j) x[j] = pk(in[2 * j], in[2 * j + 1]);
    float v = in[20];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma2(x[j], pk(v, v), x[(j + 4) & 7]);
        v = v * 0.999f;
    }
    float s = 0; for (int j = 0; j < 8; ++j) { float2 q = upk(x[j]); s += q.x + q.y; }
    if (s == 1234.5f) out[0] = s;
}
// mixed: FFMA2 (uniform) + one LDS.128 per 4 FFMA2 (the conv inner loop's ratio)
__global__ void __launch_bounds__(256) k_ffma2_lds(float* out, const float* in, int iters, float a, float b) {
    __shared__ float4 sm[256 + 64];
    sm[threadIdx.x] = make_float4(in[0], in[1], in[2], in[3]);
    __syncthreads();
    unsigned long long x[8];
    for (int j = 0; j < 8; ++j) x[j] = pk(in[2 * j], in[2 * j + 1]);
    const unsigned long long ab = pk(a, b);
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        float4 q = sm[(idx + i) & 255];
        const unsigned long long q0 = pk(q.x, q.y), q1 = pk(q.z, q.w);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma2(j & 1 ? q1 : q0, ab, x[j]);
    }
    float s = 0; for (int j = 0; j < 8; ++j) { float2 v = upk(x[j]); s += v.x + v.y; }
    if (s == 1234.5f) out[0] = s;
}

int main() {
    float *out, *in;
    cudaMalloc(&out, 4); cudaMalloc(&in, 256);
    cudaMemset(in, 0, 256);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, iters = 20000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, double fma_per_iter, auto launch) {
        launch(); cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        const double flop = (double)blocks * 256 * iters * fma_per_iter * 2;
        printf("%-14s %8.2f TFLOP/s  (%s)\n", name, flop / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    };
    run("ffma_rrr", 16, [&] { k_rrr<<<blocks, 256>>>(out, in, iters); });
    run("ffma_rur", 16, [&] { k_rur<<<blocks, 256>>>(out, in, iters, 0.999f, 1e-3f); });
    run("ffma2_u", 16, [&] { k_ffma2_u<<<blocks, 256>>>(out, in, iters, 0.999f, 1e-3f); });
    run("ffma2_bcast", 16, [&] { k_ffma2_bc<<<blocks, 256>>>(out, in, iters); });
    run("ffma2_lds", 16, [&] { k_ffma2_lds<<<blocks, 256>>>(out, in, iters, 0.999f, 1e-3f); });
    return 0;
}

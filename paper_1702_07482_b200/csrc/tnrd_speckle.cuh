// tnrd_speckle.cuh -- L-look amplitude speckle on the GPU (SURVEY §8(f)
// rank 3: the step before the despeckling path for large scenes).
//
// Reference semantics (speckle.py:51-70): n = sqrt(G / L), G ~ Gamma(L, 1)
// per pixel (so n^2 ~ Gamma(L, 1/L), E[n^2] = 1, n ~ Nakagami(L, 1)), and
// noisy = clean * n.  The reference draws G with numpy's
// Generator(Philox(key=seed)).gamma, a sequential stream whose per-sample
// draw count varies (rejection sampling) -- it cannot be reproduced by a
// parallel generator, so parity here is statistical, as SURVEY §8(f) says.
//
// Generator: counter-based Philox4x32-10 (Salmon et al., SC'11; the
// Random123 round constants and key schedule -- pinned to the published
// known-answer vector and to curand's host Philox generator in
// tests/test_speckle_cpu.py) keyed by the 64-bit seed.  Pixel i = image*H*W
// + y*W + x draws block a = 0, 1, ... as Philox(i lo, i hi, a, 0): a
// Box-Muller pair of normals + two uniforms = two Marsaglia-Tsang attempts
// (both rejected: < 0.3% of pixels for L >= 1, so warps rarely diverge into
// a second block).  Every pixel's value is a pure function of (seed, looks,
// i): bit-reproducible for any launch geometry, batch split or stream.
//
// Gamma(L, 1): Marsaglia & Tsang (ACM TOMS 2000) -- d = L - 1/3, c =
// 1/sqrt(9d), x ~ N(0, 1), v = (1 + c x)^3, accept d v when
// log(u) < x^2/2 + d - d v + d log v.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tnrd {

struct Philox4 {
    uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

// Philox4x32 with 10 rounds (multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key
// increments 0x9E3779B9 / 0xBB67AE85)
__host__ __device__ __forceinline__ Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = Philox4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// (0, 1): the top 24 bits, centred
__host__ __device__ __forceinline__ float u01(uint32_t b) {
    return ((float)(b >> 8) + 0.5f) * (1.0f / 16777216.0f);
}

struct SpeckleArgs {
    const float* clean;  // NULL: write the field n itself
    float* out;
    int64_t ld, img_stride;
    int H, W, batch;
    uint32_t k0, k1;     // seed
    float d, c, inv_l;   // Marsaglia-Tsang constants, 1 / L
    uint32_t* status;    // optional: [1] &= ~1 non-finite clean, ~2 negative clean
};

// one Marsaglia-Tsang attempt; true (and g = Gamma(L,1)/L) on acceptance
__device__ __forceinline__ bool mt_try(const SpeckleArgs& a, float x, float u, float& g) {
    const float t = fmaf(a.c, x, 1.0f);
    if (t <= 0.0f) return false;
    const float v = t * t * t;
    if (__logf(u) < 0.5f * x * x + a.d - a.d * v + a.d * logf(v)) {
        g = a.d * v * a.inv_l;
        return true;
    }
    return false;
}

// Box-Muller pair from two uniforms (angle taken in [-pi, pi) for the fast
// sine/cosine; the sign flip keeps (cos, sin)(2 pi u2))
__device__ __forceinline__ void box_muller(uint32_t b1, uint32_t b2, float& n0, float& n1) {
    const float rad = sqrtf(-2.0f * __logf(u01(b1)));
    const float th = fmaf(6.283185307179586f, u01(b2), -3.141592653589793f);
    float s, c;
    __sincosf(th, &s, &c);
    n0 = -rad * c;
    n1 = -rad * s;
}

// Gamma(L, 1)/L of pixel i
__device__ __forceinline__ float gamma_px(const SpeckleArgs& a, uint64_t i) {
    for (uint32_t att = 0;; ++att) {
        const Philox4 r = philox4x32_10(Philox4{(uint32_t)i, (uint32_t)(i >> 32), att, 0u}, a.k0, a.k1);
        float n0, n1, g;
        box_muller(r.x, r.y, n0, n1);
        if (mt_try(a, n0, u01(r.z), g)) return g;
        if (mt_try(a, n1, u01(r.w), g)) return g;
    }
}

// grid: x over the pixels of a row, y over rows (strided), z over images
__global__ void __launch_bounds__(256) speckle_kernel(const SpeckleArgs a) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int img = blockIdx.z;
    if (x >= a.W) return;
    uint32_t fbits = 0;
    for (int y = blockIdx.y; y < a.H; y += gridDim.y) {
        const uint64_t i = ((uint64_t)img * a.H + y) * a.W + x;
        const int64_t off = img * a.img_stride + (int64_t)y * a.ld + x;
        float v = sqrtf(gamma_px(a, i));
        if (a.clean) {
            const float c = __ldg(a.clean + off);
            if (!isfinite(c)) fbits |= 0x1u;
            else if (c < 0.0f) fbits |= 0x2u;
            v *= c;
        }
        a.out[off] = v;
    }
    if (fbits && a.status) atomicAnd(a.status + 1, ~fbits);
}

}  // namespace tnrd

// TMA 3-D box load probe: box (72, 38, 2) of a [planes][rows][72] fp32 tensor
// at a negative x start, mbarrier complete_tx; reports completion + values.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, int x, int y, int z, float* out, int* ok,
                      unsigned bytes) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                su32(sm)),
            "l"(reinterpret_cast<unsigned long long>(&map)), "r"(x), "r"(y), "r"(z), "r"(su32(&bar))
            : "memory");
    }
    unsigned done = 0;
    for (int i = 0; i < (1 << 22) && !done; ++i) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(su32(&bar)), "r"(0)
            : "memory");
    }
    if (threadIdx.x == 0) *ok = done;
    for (int i = threadIdx.x; i < (int)(bytes / 4); i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    const int W = 72, R = 46, P = 8, BX = 72, BY = 38, BZ = 2;
    int bx = argc > 1 ? atoi(argv[1]) : BX;
    int xs = argc > 2 ? atoi(argv[2]) : -3;
    std::vector<float> h((size_t)P * R * W);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float* d;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)R, (cuuint64_t)P};
    cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * R * 4};
    cuuint32_t box[3] = {(cuuint32_t)bx, BY, BZ}, es[3] = {1, 1, 1};
    CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es,
                                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d (box x %d, x start %d)\n", (int)r, bx, xs);
    unsigned bytes = bx * BY * BZ * 4;
    float* dout;
    int* dok;
    cudaMalloc(&dout, bytes);
    cudaMalloc(&dok, 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    probe<<<1, 128, bytes + 256>>>(map, xs, 5, 3, dout, dok, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    int ok = 0;
    std::vector<float> o(bytes / 4);
    cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data(), dout, bytes, cudaMemcpyDeviceToHost);
    printf("sync %s, complete %d\n", cudaGetErrorString(e), ok);
    // expected element (plane 3, row 5, col xs + i)
    int bad = 0;
    for (int zz = 0; zz < BZ; ++zz)
        for (int yy = 0; yy < BY; ++yy)
            for (int xx = 0; xx < bx; ++xx) {
                int gx = xs + xx, gy = 5 + yy, gz = 3 + zz;
                float want = (gx < 0 || gx >= W || gy >= R) ? 0.f : h[((size_t)gz * R + gy) * W + gx];
                if (o[(zz * BY + yy) * bx + xx] != want) ++bad;
            }
    printf("mismatches %d of %u\n", bad, bytes / 4);
    return 0;
}

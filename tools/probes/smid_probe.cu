// Which SM runs which CTA for a persistent grid of 2 x SMs CTAs that each
// need ~half an SM (the split kernel's assumption that CTAs c and c + SMs
// share an SM).  Prints the fraction of pairs (c, c + SMs) on the same SM.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void probe(int* smid_out, long long spin) {
    extern __shared__ float s[];
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    if (threadIdx.x == 0) smid_out[blockIdx.x] = (int)id;
    long long t0 = clock64();
    while (clock64() - t0 < spin) s[threadIdx.x] += 1.0f;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = 100 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, probe, 256, smem);
    const int G = sms * per;
    int* d;
    cudaMalloc(&d, G * sizeof(int));
    for (int rep = 0; rep < 3; ++rep) {
        probe<<<G, 256, smem>>>(d, 2000000);
        cudaDeviceSynchronize();
        std::vector<int> h(G);
        cudaMemcpy(h.data(), d, G * sizeof(int), cudaMemcpyDeviceToHost);
        int same = 0;
        std::vector<int> load(512, 0);
        for (int c = 0; c < G; ++c) load[h[c]]++;
        for (int c = 0; c + sms < G; ++c) same += h[c] == h[c + sms];
        int mx = 0, mn = 1 << 30;
        for (int i = 0; i < sms; ++i) { mx = std::max(mx, load[i]); mn = std::min(mn, load[i]); }
        printf("rep %d: G=%d per_sm=%d pairs(c,c+%d) same SM: %d / %d; CTAs per SM min %d max %d; first smids:",
               rep, G, per, sms, same, G - sms, mn, mx);
        for (int c = 0; c < 12; ++c) printf(" %d", h[c]);
        printf(" | c+%d:", sms);
        for (int c = 0; c < 12; ++c) printf(" %d", h[c + sms]);
        printf("\n");
    }
    return 0;
}

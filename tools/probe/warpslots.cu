// Which SM sub-partition (warpid % 4) does each warp of the frame kernel's
// launch shape (296 CTAs x 160 threads, 113 KB dynamic smem) land on?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int *out)
{
    extern __shared__ float sm[];
    unsigned smid, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    if ((threadIdx.x & 31) == 0) {
        int w = threadIdx.x >> 5;
        out[(blockIdx.x * 5 + w) * 2] = smid;
        out[(blockIdx.x * 5 + w) * 2 + 1] = wid;
    }
    sm[threadIdx.x] = 0;
    // stay resident a while so co-resident CTAs overlap
    long long t0 = clock64();
    while (clock64() - t0 < 2000000) {}
}
int main()
{
    int *d, h[296 * 5 * 2];
    cudaMalloc(&d, sizeof h);
    size_t smem = 113088;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<<<296, 160, smem>>>(d);
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    for (int b = 0; b < 296; b++) {
        if (h[b * 10] > 3) continue;
        printf("block %3d sm %d warps:", b, h[b * 10]);
        for (int w = 0; w < 5; w++) printf(" w%d->slot%d(smsp%d)", w, h[(b * 5 + w) * 2 + 1], h[(b * 5 + w) * 2 + 1] % 4);
        printf("\n");
    }
    return 0;
}

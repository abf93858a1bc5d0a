// cost of cudaPointerGetAttributes on pinned / pageable / device pointers
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
int main()
{
    void *pin, *dev;
    cudaHostAlloc(&pin, 1 << 20, cudaHostAllocDefault);
    cudaMalloc(&dev, 1 << 20);
    void *page = malloc(1 << 20);
    for (void *p : {pin, page, dev}) {
        cudaPointerAttributes a;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < 10000; i++) {
            cudaPointerGetAttributes(&a, p);
        }
        auto t1 = std::chrono::steady_clock::now();
        printf("type %d: %.3f us per call\n", (int)a.type, std::chrono::duration<double, std::micro>(t1 - t0).count() / 10000);
    }
    return 0;
}

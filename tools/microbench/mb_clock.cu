// mb_clock.cu -- is %clock64 one time base for all warps of an SM?  Each
// warp reads it right after a CTA barrier (tooling).
#include <cstdio>
__global__ void k(unsigned long long* out) {
    for (int rep = 0; rep < 4; ++rep) {
        __syncthreads();
        unsigned long long c;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if ((threadIdx.x & 31) == 0) out[rep * 16 + (threadIdx.x >> 5)] = c;
    }
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64 * 8);
    k<<<1, 512>>>(d);
    unsigned long long h[64];
    cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
    for (int rep = 0; rep < 4; ++rep) {
        printf("rep %d:", rep);
        for (int w = 0; w < 16; ++w) printf(" %lld", (long long)(h[rep * 16 + w] - h[rep * 16]));
        printf("\n");
    }
    return 0;
}

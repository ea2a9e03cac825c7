// mb_barmix.cu -- does a CTA barrier (bar.sync 0) wait for warps that are
// still working through named barriers (barrier.sync 1/2)?  (tooling)
#include <cstdio>
__device__ __forceinline__ unsigned long long clk() {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
    return c;
}
template <int Mode>
__global__ void k(unsigned long long* out, int spin) {
    const int w = threadIdx.x >> 5;
    unsigned long long arrive = 0, pass = 0;
    __syncthreads();
    const unsigned long long t0 = clk();
    if (Mode == 2) {  // no named barriers: warps 2-15 just spin on the clock
        if (w >= 2) {
            const unsigned long long until = t0 + (w < 8 ? 10000 : 20000);
            while (clk() < until) {}
        }
    } else if (Mode == 3) {  // named barriers with ids 5 and 6
        if (w >= 2 && w < 8) {
            for (int i = 0; i < spin; ++i) {
                if ((threadIdx.x & 31) == 0 && w == 2) __nanosleep(200);
                asm volatile("barrier.sync 5, 192;" ::: "memory");
            }
        } else if (w >= 8) {
            for (int i = 0; i < spin; ++i) {
                if ((threadIdx.x & 31) < 2 && w == 8) __nanosleep(300);
                asm volatile("barrier.sync 6, 256;" ::: "memory");
            }
        }
    } else if (w >= 2 && w < 8) {
        for (int i = 0; i < spin; ++i) {
            if ((threadIdx.x & 31) == 0 && w == 2) __nanosleep(200);
            if (Mode == 0) asm volatile("barrier.sync 1, 192;" ::: "memory");
            else asm volatile("bar.sync 1, 192;" ::: "memory");
        }
    } else if (w >= 8) {
        for (int i = 0; i < spin; ++i) {
            if ((threadIdx.x & 31) < 2 && w == 8) __nanosleep(300);
            if (Mode == 0) asm volatile("barrier.sync 2, 256;" ::: "memory");
            else asm volatile("bar.sync 2, 256;" ::: "memory");
        }
    } else if (threadIdx.x == 32) {
        __nanosleep(1000);
    }
    arrive = clk();
    __syncthreads();
    pass = clk();
    if ((threadIdx.x & 31) == 0) {
        out[w * 2] = arrive - t0;
        out[w * 2 + 1] = pass - t0;
    }
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64 * 8);
    unsigned long long h[64];
    const char* names[] = {"barrier.sync 1/2", "bar.sync 1/2", "clock spin", "barrier.sync 5/6"};
    for (int mode = 0; mode < 4; ++mode) {
        if (mode == 0) k<0><<<1, 512>>>(d, 20);
        else if (mode == 1) k<1><<<1, 512>>>(d, 20);
        else if (mode == 2) k<2><<<1, 512>>>(d, 20);
        else k<3><<<1, 512>>>(d, 20);
        cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
        printf("%s: warp arrive/pass:", names[mode]);
        for (int w = 0; w < 16; ++w) printf(" %d:%llu/%llu", w, h[2 * w], h[2 * w + 1]);
        printf("\n");
    }
    return 0;
}

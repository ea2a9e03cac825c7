// pub_check.cu -- does one thread's release (red.release.gpu / fence + st)
// after a CTA barrier publish the global stores of OTHER warps of its CTA?
// Producer CTA: warps [1, 16) write a 4 KiB node stamped with the round
// number, bar.sync, then thread 0 publishes the round through a flag
// (mode 0: red.release.gpu by thread 0; mode 1: every writer fences first,
// then thread 0 red.release; mode 2: thread 0 st.release).  Consumer CTA on
// another SM: polls the flag (ld.acquire), reads the node, counts stale
// words, then hands the token back.  Tooling.
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
    uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__global__ void __launch_bounds__(512) pub(uint32_t* node, uint32_t* flag, uint32_t* back, int rounds, int mode,
                                           unsigned long long* stale) {
    const int tid = threadIdx.x;
    if (blockIdx.x == 0) {  // producer
        for (int r = 1; r <= rounds; ++r) {
            if (tid == 0) { while (ld_acq(back) != (uint32_t)(r - 1)) {} }
            __syncthreads();
            if (mode >= 3) {
                // named barrier over warps 0..7 only: warps 4..7 write, thread 0 releases
                if (tid < 256) {
                    if (tid >= 128) for (int i = tid - 128; i < 1024; i += 128) __stcg(node + i, (uint32_t)r);
                    if (mode == 4) asm volatile("bar.sync 1, 256;" ::: "memory");
                    else asm volatile("barrier.sync 1, 256;" ::: "memory");
                    if (tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
                }
                continue;
            }
            if (tid >= 32) {
                for (int i = tid - 32; i < 1024; i += 480) __stcg(node + i, (uint32_t)r);
                if (mode == 1) __threadfence();
            }
            __syncthreads();
            if (tid == 0) {
                if (mode == 2) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"((uint32_t)r) : "memory");
                else asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
            }
        }
    } else if (blockIdx.x == gridDim.x - 1) {  // consumer, far SM
        __shared__ uint32_t go;
        unsigned long long bad = 0;
        for (int r = 1; r <= rounds; ++r) {
            if (tid == 0) { while (ld_acq(flag) != (uint32_t)r) {} go = r; }
            __syncthreads();
            for (int i = tid; i < 1024; i += 512) bad += __ldcg(node + i) != (uint32_t)r;
            __syncthreads();
            if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(back), "r"((uint32_t)r) : "memory");
        }
        atomicAdd(stale, bad);
    }
}

int main() {
    uint32_t *node, *flag, *back; unsigned long long* stale;
    CK(cudaMalloc(&node, 4096)); CK(cudaMalloc(&flag, 256)); CK(cudaMalloc(&back, 256)); CK(cudaMalloc(&stale, 8));
    for (int mode = 0; mode < 5; ++mode) {
        for (int far = 2; far <= 148; far += 73) {
            CK(cudaMemset(node, 0, 4096)); CK(cudaMemset(flag, 0, 256)); CK(cudaMemset(back, 0, 256)); CK(cudaMemset(stale, 0, 8));
            const int rounds = 200000;
            pub<<<far, 512>>>(node, flag, back, rounds, mode, stale);
            CK(cudaDeviceSynchronize());
            unsigned long long s; CK(cudaMemcpy(&s, stale, 8, cudaMemcpyDeviceToHost));
            printf("mode %d (%s) grid %3d: %llu stale words in %d rounds\n", mode,
                   mode == 0 ? "writers no fence, t0 red.release" : mode == 1 ? "writers fence, t0 red.release" : mode == 2 ? "writers no fence, t0 st.release" : mode == 3 ? "named barrier.sync 1,256, t0 red.release" : "named bar.sync 1,256, t0 red.release",
                   far, s, rounds);
        }
    }
    return 0;
}

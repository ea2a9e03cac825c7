// mb_sync.cu -- cost of the CTA synchronisation primitives the three-level
// delete server uses (tooling): SM cycles per operation, one CTA.
#include <cstdio>
#include <cstdlib>
#include "../../paper_1906_06504_b200/csrc/bh_device.cuh"
using namespace bh;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long clk() {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
    return c;
}

// mode 0: try_wait on a completed mbarrier phase
// mode 1: mbarrier arrive (release.cta) with no stores outstanding
// mode 2: 4 KiB of st.global.cg by the warp, then arrive (release.cta)
// mode 3: 4 KiB of st.global.cg by the warp, then arrive.relaxed
// mode 4: named barrier (12 warps), no stores
// mode 5: named barrier (12 warps) after 4 KiB st.global.cg per group of 4 warps
// mode 6: clock read right after 4 KiB st.global.cg
__global__ void sync_bench(int mode, int iters, unsigned long long* out, uint4* g) {
    __shared__ __align__(8) unsigned long long mb[2];
    __shared__ unsigned long long flag;
    if (threadIdx.x == 0) flag = 0;
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { mb_init(&mb[0], 1); mb_init(&mb[1], 1); }
    __syncthreads();
    if (threadIdx.x == 0) mb_arrive(&mb[0]);  // phase 0 of mb[0] complete
    __syncthreads();
    unsigned long long t0 = clk(), acc = 0;
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
            if (w == 0) mb_wait(&mb[0], 0);
        } else if (mode == 1 || mode == 2 || mode == 3) {
            if (w == 0) {
                if (mode >= 2)
                    for (int i = lane; i < 256; i += 32) __stcg(g + i + 256 * (it & 7), make_uint4(it, 1, 2, 3));
                __syncwarp();
                if (lane == 0) {
                    if (mode == 3) asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&mb[1])) : "memory");
                    else mb_arrive(&mb[1]);
                }
                __syncwarp();
            }
        } else if (mode == 4 || mode == 5) {
            if (w < 12) {
                if (mode == 5 && (w & 3) == 0)
                    for (int i = lane; i < 256; i += 32) __stcg(g + i + 256 * (w >> 2), make_uint4(it, 1, 2, 3));
                asm volatile("barrier.sync 6, 384;" ::: "memory");
            }
        } else if (mode == 7) {  // bar.sync (aligned) x12 warps
            if (w < 12) asm volatile("bar.sync 6, 384;" ::: "memory");
        } else if (mode == 8) {  // __syncthreads (all 16 warps)
            __syncthreads();
        } else if (mode == 9) {  // volatile smem flag already set + fence.cta
            if (w == 0) {
                volatile unsigned long long* f = &flag;
                while (*f != 0) {}
                __threadfence_block();
            }
        } else if (mode == 10) {  // mbarrier test_wait on a completed phase
            if (w == 0) acc += mb_test(&mb[0], 0);
        } else if (mode == 11) {  // __threadfence with no stores outstanding
            if (w == 0) __threadfence();
        } else if (mode == 12) {  // 4 KiB st.cg by the warp, then __threadfence by lane 0
            if (w == 0) {
                for (int i = lane; i < 256; i += 32) __stcg(g + i + 256 * (it & 7), make_uint4(it, 1, 2, 3));
                __syncwarp();
                if (lane == 0) __threadfence();
                __syncwarp();
            }
        } else if (mode == 13) {  // 4 KiB st.cg by 8 warps, CTA barrier, __threadfence by thread 0
            if (w < 8)
                for (int i = threadIdx.x; i < 256; i += 256) __stcg(g + i + 256 * (it & 7), make_uint4(it, 1, 2, 3));
            __syncthreads();
            if (threadIdx.x == 0) __threadfence();
            __syncthreads();
        } else if (mode == 6) {
            if (w == 0) {
                for (int i = lane; i < 256; i += 32) __stcg(g + i, make_uint4(it, 1, 2, 3));
                acc += clk();
            }
        }
    }
    unsigned long long t1 = clk();
    if (threadIdx.x == 0) out[mode] = (t1 - t0) / iters + (acc == 1 ? 1 : 0);
}

int main() {
    unsigned long long* o;
    uint4* g;
    CK(cudaMalloc(&o, 16 * 8));
    CK(cudaMalloc(&g, 4096 * 8));
    const char* names[] = {"try_wait on a completed phase", "arrive.release, no stores", "4 KiB st.cg + arrive.release",
                           "4 KiB st.cg + arrive.relaxed", "named barrier x12 warps", "named barrier after 4 KiB st.cg",
                           "4 KiB st.cg + clock read", "bar.sync (aligned) x12 warps", "__syncthreads x16 warps",
                           "volatile smem flag (set) + fence.cta", "test_wait on a completed phase",
                           "__threadfence, nothing outstanding", "4 KiB st.cg + __threadfence (warp)",
                           "4 KiB st.cg (8 warps) + bar + fence + bar"};
    for (int m = 0; m <= 13; ++m) {
        sync_bench<<<1, 512>>>(m, 2000, o, g);
        CK(cudaDeviceSynchronize());
        unsigned long long c;
        CK(cudaMemcpy(&c, o + m, 8, cudaMemcpyDeviceToHost));
        printf("sync %-36s : %llu cycles/iter\n", names[m], c);
    }
    return 0;
}

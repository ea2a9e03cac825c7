// mb_sort.cu -- sort_batch of one K-key batch by one CTA (tooling): the
// shared-memory bitonic network with a CTA barrier per stage
// (cta_bitonic_sort, the round-1 kernel) against the register network
// (cta_sort_batch: in-register / shuffle stages, shared memory only for
// strides >= 32E).  SM cycles per sort, global batch -> sorted in smem.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include "../../paper_1906_06504_b200/csrc/bh_device.cuh"
using namespace bh;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

template <typename Key, int K, int T, bool Reg>
__global__ void __launch_bounds__(T) sort_bench(const Key* in, int iters, unsigned long long* out, Key* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    Key* s0 = reinterpret_cast<Key*>(sm);
    Key* s1 = s0 + K;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
    for (int it = 0; it < iters; ++it) {
        const Key* g = in + (it & 7) * K;
        if constexpr (Reg) {
            cta_sort_batch<Key, K, T>(g, K, s0, s1);
        } else {
            for (uint32_t i = threadIdx.x; i < (uint32_t)K; i += T) s0[i] = g[i];
            __syncthreads();
            cta_bitonic_sort<Key, K, T>(s0);
        }
        if (threadIdx.x == 0) sink[it & 7] = s0[K / 2];
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    for (int i = threadIdx.x; i < K; i += T) sink[8 + i] = s0[i];
}

template <typename Key, int K, int T, bool Reg>
void run(const char* kname) {
    std::mt19937_64 rng(7);
    std::vector<Key> h(8 * K);
    for (auto& x : h) x = (Key)(rng() >> 8) & (Key)~(Key)0 >> 1;
    Key *d, *sink;
    unsigned long long* o;
    CK(cudaMalloc(&d, 8 * K * sizeof(Key)));
    CK(cudaMalloc(&sink, (8 + K) * sizeof(Key)));
    CK(cudaMalloc(&o, 8));
    CK(cudaMemcpy(d, h.data(), 8 * K * sizeof(Key), cudaMemcpyHostToDevice));
    auto kern = sort_bench<Key, K, T, Reg>;
    const int smem = 2 * K * sizeof(Key);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, T, smem>>>(d, 1, o, sink);
    CK(cudaDeviceSynchronize());
    std::vector<Key> got(K);
    CK(cudaMemcpy(got.data(), sink + 8, K * sizeof(Key), cudaMemcpyDeviceToHost));
    std::vector<Key> ref(h.begin(), h.begin() + K);
    std::sort(ref.begin(), ref.end());
    const bool ok = got == ref;
    kern<<<1, T, smem>>>(d, 2000, o, sink);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("sort %-4s K=%-5d T=%-4d %-9s : %6llu cycles %s\n", kname, K, T, Reg ? "register" : "smem", c,
           ok ? "" : "WRONG");
    cudaFree(d); cudaFree(sink); cudaFree(o);
}

int main() {
    run<uint32_t, 256, 128, false>("u32");  run<uint32_t, 256, 128, true>("u32");
    run<uint32_t, 512, 256, false>("u32");  run<uint32_t, 512, 256, true>("u32");
    run<uint32_t, 1024, 512, false>("u32"); run<uint32_t, 1024, 512, true>("u32");
    run<uint32_t, 2048, 512, false>("u32"); run<uint32_t, 2048, 512, true>("u32");
    run<unsigned long long, 256, 128, false>("u64");  run<unsigned long long, 256, 128, true>("u64");
    run<unsigned long long, 1024, 512, false>("u64"); run<unsigned long long, 1024, 512, true>("u64");
    run<unsigned long long, 2048, 512, false>("u64"); run<unsigned long long, 2048, 512, true>("u64");
    return 0;
}

// mb_round.cu -- cost of one merge "round" of the three-level delete server
// on a 512-thread CTA (tooling): G concurrent half merges of two K=1024 u32
// batches, each by NW warps (the product's grp_merge_half), followed by a
// named barrier over the merge warps; SM cycles per round.
//
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../../include mb_round.cu -o mb_round
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

#include "../../paper_1906_06504_b200/csrc/bh_select.cuh"

using namespace bh;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

constexpr int K = 1024;

// Noise (warps 0-1 while the merges run): 0 none; 1 warp 0 stores 4 KiB to
// global and fences (__threadfence) in a loop; 2 warp 1 polls a global word
// with ld.acquire.gpu; 3 warp 1 relaxed polls + fence.acq_rel on each
template <int NW, int G, bool Inl, int Noise>
__global__ void __launch_bounds__(512, 1) round_bench(const uint32_t* in, int iters, unsigned long long* out, uint32_t* sink,
                                                       uint32_t* scratch, volatile uint32_t* stop) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint32_t* A = reinterpret_cast<uint32_t*>(sm);
    uint32_t* B = A + K;
    uint32_t* H = B + K;  // G outputs
    for (int i = threadIdx.x; i < 2 * K; i += 512) A[i] = in[i];
    __syncthreads();
    const uint32_t w = threadIdx.x >> 5;
    const uint32_t mw = w - 2;  // merge warps 2..
    constexpr uint32_t kMergeThreads = 32 * NW * G;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
    if (w == 0 && Noise == 1) {
        uint4 v = make_uint4(1, 2, 3, 4);
        while (!*stop) {
            for (int i = threadIdx.x; i < 256; i += 32) __stcg(reinterpret_cast<uint4*>(scratch) + i, v);
            __threadfence();
            v.x++;
        }
    }
    if (w == 1 && (Noise == 2 || Noise == 3)) {
        uint32_t acc = 0;
        while (!*stop) {
            uint32_t x;
            if (Noise == 2) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(scratch + 1024) : "memory");
            else {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(scratch + 1024) : "memory");
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
            acc += x;
        }
        if (acc == 12345) sink[0] = acc;
    }
    if (w >= 2 && mw < (uint32_t)(NW * G)) {
        for (int it = 0; it < iters; ++it) {
            const uint32_t g = mw / NW;
            if (g & 1)
                grp_merge_half<uint32_t, K, NW, true, false, Inl>(A, B, H + g * K, mw % NW);
            else
                grp_merge_half<uint32_t, K, NW, false, false, Inl>(A, B, H + g * K, mw % NW);
            asm volatile("barrier.sync 6, %0;" ::"r"(kMergeThreads) : "memory");
        }
    }
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
    if (threadIdx.x == 64) {
        out[0] = (t1 - t0) / iters;
        *stop = 1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += 512) sink[i] = H[i];
}

// I-cache pressure: C distinct inlined copies of the merge, round r runs copy
// r % C (the kernel's server inlines a copy per call site).
template <int C>
struct Copies {
    static __device__ __forceinline__ void run(int r, const uint32_t* A, const uint32_t* B, uint32_t* H, uint32_t mw) {
        if (r % (C + 1) == C) {
            if (C & 1) grp_merge_half<uint32_t, K, 4, true, false, true>(A, B, H, mw);
            else grp_merge_half<uint32_t, K, 4, false, false, true>(A, B, H, mw);
            asm volatile("" ::"n"(C));
        } else {
            Copies<C - 1>::run(r, A, B, H, mw);
        }
    }
};
template <>
struct Copies<0> {
    static __device__ __forceinline__ void run(int, const uint32_t* A, const uint32_t* B, uint32_t* H, uint32_t mw) {
        grp_merge_half<uint32_t, K, 4, false, false, true>(A, B, H, mw);
    }
};
template <int C>
__global__ void __launch_bounds__(512, 1) icache_bench(const uint32_t* in, int iters, unsigned long long* out, uint32_t* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint32_t* A = reinterpret_cast<uint32_t*>(sm);
    uint32_t* B = A + K;
    uint32_t* H = B + K;
    for (int i = threadIdx.x; i < 2 * K; i += 512) A[i] = in[i];
    __syncthreads();
    const uint32_t w = threadIdx.x >> 5;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
    if (w >= 2 && w < 6) {
        for (int it = 0; it < iters; ++it) {
            Copies<C>::run(it % (C + 1) + 0 * it, A, B, H, w - 2);
            asm volatile("barrier.sync 6, 128;" ::: "memory");
        }
    }
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
    if (threadIdx.x == 64) out[0] = (t1 - t0) / iters;
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += 512) sink[i] = H[i];
}
template <int C>
void run_icache() {
    std::vector<uint32_t> h(2 * K);
    std::mt19937 rng(1);
    for (auto& x : h) x = rng() >> 1;
    std::sort(h.begin(), h.begin() + K);
    std::sort(h.begin() + K, h.end());
    uint32_t *d, *sink;
    unsigned long long* o;
    CK(cudaMalloc(&d, 2 * K * 4));
    CK(cudaMalloc(&sink, K * 4));
    CK(cudaMalloc(&o, 8));
    CK(cudaMemcpy(d, h.data(), 2 * K * 4, cudaMemcpyHostToDevice));
    auto kern = icache_bench<C>;
    const int smem = 3 * K * 4 + 64;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, 512, smem>>>(d, 4000, o, sink);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("icache copies=%d : %llu cycles per round\n", C + 1, c);
    cudaFree(d); cudaFree(sink); cudaFree(o);
}

template <int NW, int G, bool Inl, int Noise = 0>
void run(const char* name) {
    std::mt19937 rng(1);
    std::vector<uint32_t> h(2 * K);
    for (auto& x : h) x = rng() >> 1;
    std::sort(h.begin(), h.begin() + K);
    std::sort(h.begin() + K, h.end());
    uint32_t *d, *sink;
    unsigned long long* o;
    CK(cudaMalloc(&d, 2 * K * 4));
    CK(cudaMalloc(&sink, K * 4));
    CK(cudaMalloc(&o, 8));
    CK(cudaMemcpy(d, h.data(), 2 * K * 4, cudaMemcpyHostToDevice));
    auto kern = round_bench<NW, G, Inl, Noise>;
    uint32_t* scratch;
    uint32_t* stop;
    CK(cudaMalloc(&scratch, 8192));
    CK(cudaMalloc(&stop, 4));
    CK(cudaMemset(scratch, 0, 8192));
    const int smem = (2 + G) * K * 4 + 64;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaMemset(stop, 0, 4));
    kern<<<1, 512, smem>>>(d, 1, o, sink, scratch, stop);
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> got(K), ref(2 * K);
    CK(cudaMemcpy(got.data(), sink, K * 4, cudaMemcpyDeviceToHost));
    std::merge(h.begin(), h.begin() + K, h.begin() + K, h.end(), ref.begin());
    if (!std::equal(got.begin(), got.end(), ref.begin())) printf("%s WRONG OUTPUT\n", name);
    CK(cudaMemset(stop, 0, 4));
    kern<<<1, 512, smem>>>(d, 4000, o, sink, scratch, stop);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("round %-10s NW=%d G=%d inline=%d noise=%d : %llu cycles\n", name, NW, G, (int)Inl, Noise, c);
    cudaFree(d); cudaFree(sink); cudaFree(o);
}

// The server's round shape: three groups of 4 warps, each merging its own
// pair of buffers with the run-time variant (grp_merge_half_rt); group 2
// writes its half to global memory when Glob.
template <bool Glob, int Live = 0>
__global__ void __launch_bounds__(512, 1) rt_bench(const uint32_t* in, int iters, unsigned long long* out, uint32_t* sink, uint32_t* gout,
                                                    volatile uint32_t* stop = nullptr) {
    extern __shared__ __align__(16) unsigned char sm[];
    if (blockIdx.x > 0) {  // the other CTAs: wait like queued heap CTAs (one lane polls, the rest at a barrier)
        if (threadIdx.x == 0) {
            uint32_t n = 0;
            while (!*stop) { if (++n > 32) __nanosleep(64); }
        }
        __syncthreads();
        return;
    }
    uint32_t* bufs = reinterpret_cast<uint32_t*>(sm);  // 9 buffers: 3 x (A, B, H)
    for (int i = threadIdx.x; i < 2 * K; i += 512) {
        bufs[i] = in[i];
        bufs[3 * K + i] = in[i];
        bufs[6 * K + i] = in[i];
    }
    __syncthreads();
    const uint32_t w = threadIdx.x >> 5;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
    if (w >= 2 && w < 14) {
        const uint32_t mw = w - 2, grp = mw >> 2, gw = mw & 3;
        // Live: values kept live across the merges (register pressure of the
        // server's op loop)
        uint32_t live[Live > 0 ? Live : 1];
#pragma unroll
        for (int q = 0; q < Live; ++q) live[q] = in[q] * (threadIdx.x + q);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < Live; ++q) asm volatile("" : "+r"(live[q]));
            const uint32_t* A = bufs + 3 * K * grp;
            const uint32_t* B = A + K;
            uint32_t* o = bufs + 3 * K * grp + 2 * K;
            bool glob = false;
            if (Glob && grp == 2) { o = gout; glob = true; }
            grp_merge_half_rt<uint32_t, K, 4>(A, B, o, gw, grp == 1, glob);
            asm volatile("barrier.sync 6, 384;" ::: "memory");
        }
        uint32_t acc = 0;
#pragma unroll
        for (int q = 0; q < Live; ++q) acc += live[q];
        if (acc == 0x12345) sink[0] = acc;
    }
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
    if (threadIdx.x == 64) {
        out[0] = (t1 - t0) / iters;
        if (stop) *stop = 1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += 512) sink[i] = bufs[2 * K + i];
}
template <bool Glob, int Live = 0>
void run_rt(int grid = 1) {
    std::vector<uint32_t> h(2 * K);
    std::mt19937 rng(1);
    for (auto& x : h) x = rng() >> 1;
    std::sort(h.begin(), h.begin() + K);
    std::sort(h.begin() + K, h.end());
    uint32_t *d, *sink, *gout;
    unsigned long long* o;
    CK(cudaMalloc(&d, 2 * K * 4));
    CK(cudaMalloc(&sink, K * 4));
    CK(cudaMalloc(&gout, K * 4));
    CK(cudaMalloc(&o, 8));
    CK(cudaMemcpy(d, h.data(), 2 * K * 4, cudaMemcpyHostToDevice));
    auto kern = rt_bench<Glob, Live>;
    const int smem = 9 * K * 4 + 64;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    uint32_t* stop;
    CK(cudaMalloc(&stop, 4));
    CK(cudaMemset(stop, 0, 4));
    kern<<<grid, 512, smem>>>(d, 4000, o, sink, gout, stop);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> got(K), ref(2 * K);
    CK(cudaMemcpy(got.data(), sink, K * 4, cudaMemcpyDeviceToHost));
    std::merge(h.begin(), h.begin() + K, h.begin() + K, h.end(), ref.begin());
    printf("rt round (3 groups, own buffers, global=%d, grid %d, live %d): %llu cycles %s\n", (int)Glob, grid, Live, c,
           std::equal(got.begin(), got.end(), ref.begin()) ? "" : "WRONG");
}

int main() {
    run_rt<false>();
    run_rt<true>();
    run_rt<false, 40>();
    run_rt<false, 60>();
    run_rt<false, 75>();
    run_rt<false, 90>();
    run_icache<0>();
    run_icache<3>();
    run_icache<11>();
    run_icache<23>();
    run<4, 1, true>("bt");
    run<4, 1, false>("bt");
    run<4, 2, true>("bt");
    run<4, 3, true>("bt");
    run<2, 1, true>("bt");
    run<2, 6, true>("bt");
    run<8, 1, true>("bt");
    run<8, 1, false>("bt");
    run<4, 1, true, 1>("bt");
    run<4, 3, true, 1>("bt");
    run<4, 1, true, 2>("bt");
    run<4, 3, true, 2>("bt");
    run<4, 1, true, 3>("bt");
    run<4, 3, true, 3>("bt");
    return 0;
}

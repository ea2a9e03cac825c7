// mb.cu -- latency microbenchmarks of the heap's CTA primitives on one B200
// (tooling, not product code).  Each test prints SM cycles per operation.
//
//   make -C tools/microbench && tools/microbench/mb
//
//  merge   : cta_merge_full (2K -> hi/lo) and variants, one CTA, smem only
//  sort    : cta_bitonic_sort of K keys
//  handoff : a 4 KiB node passed between two CTAs on different SMs through a
//            versioned state word (write, barrier, release / poll, claim+load)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <string>

#include "../../paper_1906_06504_b200/csrc/bh_device.cuh"
#include "mb_variants.cuh"

using namespace bh;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

// Padded layout: element i lives at i + i/32 (one pad word per 32), so
// split-search probes at power-of-two strides fall in different banks.
__device__ __forceinline__ uint32_t padi(uint32_t i) { return i + (i >> 5); }

template <typename Key, int K, int P>
__device__ __forceinline__ void half_pad(const Key* A, const Key* B, Key* out) {
    const uint32_t t0 = threadIdx.x * P;
    if (t0 >= (uint32_t)K) return;
    const uint32_t d = t0;
    const uint32_t lo = 0, hi = d < K ? d : K;
    uint32_t base = lo;
#pragma unroll
    for (uint32_t step = (uint32_t)K; step > 0; step >>= 1) {
        const uint32_t p = base + step;
        if (p <= hi && A[padi(p - 1)] <= B[padi(d - p)]) base = p;
    }
    const uint32_t i = base, j = d - base;
    Key a[P + 1], b[P + 1];
#pragma unroll
    for (int e = 0; e < P; ++e) {
        a[e] = i + e < K ? A[padi(i + e)] : KeyLimits<Key>::kMax;
        b[e] = j + e < K ? B[padi(j + e)] : KeyLimits<Key>::kMax;
    }
    a[P] = b[P] = KeyLimits<Key>::kMax;
    uint32_t ra = K - i, rb = K - j;
    Key o[P];
#pragma unroll
    for (int e = 0; e < P; ++e) {
        const bool ta = rb == 0 || (ra != 0 && a[0] <= b[0]);
        o[e] = ta ? a[0] : b[0];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            a[q] = ta ? a[q + 1] : a[q];
            b[q] = ta ? b[q] : b[q + 1];
        }
        ra -= ta;
        rb -= !ta;
    }
#pragma unroll
    for (int e = 0; e < P; ++e) out[padi(t0 + e)] = o[e];
}

template <typename Key, int K, int T, int P>
__global__ void __launch_bounds__(T) halfpad_bench(const Key* in, int iters, unsigned long long* out, Key* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr int KP = K + K / 32;
    Key* A = reinterpret_cast<Key*>(sm);
    Key* B = A + KP;
    Key* H = B + KP;
    for (int i = threadIdx.x; i < K; i += T) { A[padi(i)] = in[i]; B[padi(i)] = in[K + i]; }
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        half_pad<Key, K, P>(A, B, H);
        __syncthreads();
        if (threadIdx.x == 0) A[0] = H[0] < A[0] ? H[0] : A[0];
        __syncthreads();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    for (int i = threadIdx.x; i < K; i += T) sink[i] = H[padi(i)];
}

template <int K, int T, int P>
void run_halfpad(const char* name) {
    using Key = uint32_t;
    std::mt19937 rng(1);
    std::vector<Key> h(2 * K);
    for (auto& x : h) x = rng() >> 1;
    std::sort(h.begin(), h.begin() + K);
    std::sort(h.begin() + K, h.end());
    Key *d, *sink;
    unsigned long long* o;
    CK(cudaMalloc(&d, 2 * K * 4));
    CK(cudaMalloc(&sink, 2 * K * 4 + 16));
    CK(cudaMalloc(&o, 8 * 8));
    CK(cudaMemcpy(d, h.data(), 2 * K * 4, cudaMemcpyHostToDevice));
    auto kern = halfpad_bench<Key, K, T, P>;
    const int smem = 3 * (K + K / 32) * 4 + 64;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, T, smem>>>(d, 1, o, sink);
    CK(cudaDeviceSynchronize());
    std::vector<Key> got(K), ref(2 * K);
    CK(cudaMemcpy(got.data(), sink, K * 4, cudaMemcpyDeviceToHost));
    std::merge(h.begin(), h.begin() + K, h.begin() + K, h.end(), ref.begin());
    if (!std::equal(got.begin(), got.end(), ref.begin())) printf("halfpad %s WRONG OUTPUT\n", name);
    kern<<<1, T, smem>>>(d, 2000, o, sink);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("halfpad %-20s K=%d T=%d P=%d : %llu cycles\n", name, K, T, P, c);
    cudaFree(d); cudaFree(sink); cudaFree(o);
}

// Half-merge variants: P outputs per thread, binary (Q=0) or quaternary (Q=1)
// split search.
template <typename Key, int K, int P, int Q>
__device__ __forceinline__ void half_var(const Key* A, const Key* B, Key* out) {
    const uint32_t t0 = threadIdx.x * P;
    if (t0 >= (uint32_t)K) return;
    uint32_t i;
    if constexpr (Q) i = split_q<Key, Pow4Floor<K>::v>(A, B, t0, K, K);
    else i = merge_split<Key, K>(A, B, t0, K, K);
    Key run[P];
    merge_window<Key, P>(A, i, K, B, t0 - i, K, run);
    store_run<Key, P>(out + t0, run);
}

template <typename Key, int K, int T, int P, int Q>
__global__ void __launch_bounds__(T) half_bench(const Key* in, int iters, unsigned long long* out, Key* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    Key* A = reinterpret_cast<Key*>(sm);
    Key* B = A + K;
    Key* H = B + K;
    for (int i = threadIdx.x; i < 2 * K; i += T) A[i] = in[i];
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        half_var<Key, K, P, Q>(A, B, H);
        __syncthreads();
        if (threadIdx.x == 0) A[0] = H[0] < A[0] ? H[0] : A[0];
        __syncthreads();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    for (int i = threadIdx.x; i < K; i += T) sink[i] = H[i];
}

template <int K, int T, int P, int Q>
void run_half(const char* name) {
    using Key = uint32_t;
    std::mt19937 rng(1);
    std::vector<Key> h(2 * K);
    for (auto& x : h) x = rng() >> 1;
    std::sort(h.begin(), h.begin() + K);
    std::sort(h.begin() + K, h.end());
    Key *d, *sink;
    unsigned long long* o;
    CK(cudaMalloc(&d, 2 * K * 4));
    CK(cudaMalloc(&sink, 2 * K * 4 + 16));
    CK(cudaMalloc(&o, 8 * 8));
    CK(cudaMemcpy(d, h.data(), 2 * K * 4, cudaMemcpyHostToDevice));
    auto kern = half_bench<Key, K, T, P, Q>;
    const int smem = 3 * K * 4 + 64;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, T, smem>>>(d, 1, o, sink);
    CK(cudaDeviceSynchronize());
    std::vector<Key> got(K), ref(2 * K);
    CK(cudaMemcpy(got.data(), sink, K * 4, cudaMemcpyDeviceToHost));
    std::merge(h.begin(), h.begin() + K, h.begin() + K, h.end(), ref.begin());
    if (!std::equal(got.begin(), got.end(), ref.begin())) printf("half %s WRONG OUTPUT\n", name);
    kern<<<1, T, smem>>>(d, 2000, o, sink);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("half  %-22s K=%d T=%d P=%d : %llu cycles\n", name, K, T, P, c);
    cudaFree(d); cudaFree(sink); cudaFree(o);
}

// Warp-tile bitonic half merge (candidate for the product): each warp owns a
// tile of 32E consecutive outputs [D, D + 32E) of merge(A, B).  (1) The
// merge-path split of diagonal D by a fixed-trip 32-ary search (lane l tests
// lo + (l+1)g with an odd stride g, ballot + popc; two rounds for K <= 1024).
// (2) The tile = the 32E smallest of the windows A[a, a+32E) and B[b, b+32E)
// (sentinel past the ends): min(Aw[i], Bw[32E-1-i]) is bitonic and holds
// exactly them.  (3) A bitonic half-cleaner network sorts it: strides >= 32
// in registers, below with shuffles.  Lane l ends with outputs D + 32e + l.
template <typename Key, int K, int E>
__device__ __forceinline__ void warp_half_bt(const Key* __restrict__ A, const Key* __restrict__ B,
                                             Key* __restrict__ out, uint32_t D) {
    constexpr uint32_t W = 32u * E;
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t lo = D > (uint32_t)K ? D - K : 0u;
    uint32_t hi = D < (uint32_t)K ? D : (uint32_t)K;
    // fixed trips: each round shrinks the range by 32
#pragma unroll
    for (uint32_t span = (uint32_t)K; span > 0; span >>= 5) {
        const uint32_t g = span > 32 ? ((span + 31u) >> 5) | 1u : 1u;
        const uint32_t p = lo + (lane + 1u) * g;
        const bool ok = p <= hi && A[p - 1] <= B[D - p];
        const uint32_t c = __popc(__ballot_sync(0xFFFFFFFFu, ok));
        lo += c * g;
        const uint32_t h2 = lo + g - 1u;
        hi = h2 < hi ? h2 : hi;
        if (g == 1u) break;
    }
    const uint32_t a = lo, b = D - lo;
    Key v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const uint32_t i = e * 32u + lane;
        const Key x = a + i < (uint32_t)K ? A[a + i] : KeyLimits<Key>::kMax;
        const uint32_t j = b + (W - 1u - i);
        const Key y = j < (uint32_t)K ? B[j] : KeyLimits<Key>::kMax;
        v[e] = x < y ? x : y;
    }
#pragma unroll
    for (int rs = E / 2; rs >= 1; rs >>= 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e & rs) == 0) {
                const Key x = v[e], y = v[e + rs];
                v[e] = x < y ? x : y;
                v[e + rs] = x < y ? y : x;
            }
        }
    }
#pragma unroll
    for (int ls = 16; ls >= 1; ls >>= 1) {
        const bool upper = (lane & ls) != 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const Key o = __shfl_xor_sync(0xFFFFFFFFu, v[e], ls);
            v[e] = upper ? (v[e] < o ? o : v[e]) : (v[e] < o ? v[e] : o);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) out[D + e * 32u + lane] = v[e];
}

template <typename Key, int K, int T, int E>
__global__ void __launch_bounds__(T) halfbt_bench(const Key* in, int iters, unsigned long long* out, Key* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    Key* A = reinterpret_cast<Key*>(sm);
    Key* B = A + K;
    Key* H = B + K;
    for (int i = threadIdx.x; i < 2 * K; i += T) A[i] = in[i];
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (uint32_t D = (threadIdx.x >> 5) * 32u * E; D < (uint32_t)K; D += (T / 32) * 32u * E)
            warp_half_bt<Key, K, E>(A, B, H, D);
        __syncthreads();
        if (threadIdx.x == 0) A[0] = H[0] < A[0] ? H[0] : A[0];
        __syncthreads();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    for (int i = threadIdx.x; i < K; i += T) sink[i] = H[i];
}

template <int K, int T, int E>
void run_halfbt(const char* name) {
    using Key = uint32_t;
    std::mt19937 rng(1);
    std::vector<Key> h(2 * K);
    for (auto& x : h) x = rng() >> 1;
    std::sort(h.begin(), h.begin() + K);
    std::sort(h.begin() + K, h.end());
    Key *d, *sink;
    unsigned long long* o;
    CK(cudaMalloc(&d, 2 * K * 4));
    CK(cudaMalloc(&sink, 2 * K * 4 + 16));
    CK(cudaMalloc(&o, 8 * 8));
    CK(cudaMemcpy(d, h.data(), 2 * K * 4, cudaMemcpyHostToDevice));
    auto kern = halfbt_bench<Key, K, T, E>;
    const int smem = 3 * K * 4 + 64;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, T, smem>>>(d, 1, o, sink);
    CK(cudaDeviceSynchronize());
    std::vector<Key> got(K), ref(2 * K);
    CK(cudaMemcpy(got.data(), sink, K * 4, cudaMemcpyDeviceToHost));
    std::merge(h.begin(), h.begin() + K, h.begin() + K, h.end(), ref.begin());
    if (!std::equal(got.begin(), got.end(), ref.begin())) printf("halfbt %s WRONG OUTPUT\n", name);
    kern<<<1, T, smem>>>(d, 2000, o, sink);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("halfbt %-21s K=%d T=%d E=%d : %llu cycles\n", name, K, T, E, c);
    cudaFree(d); cudaFree(sink); cudaFree(o);
}

template <typename Key, int K, int T, int V>
__global__ void __launch_bounds__(T) merge_bench(const Key* in, int iters, unsigned long long* out, Key* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    Key* A = reinterpret_cast<Key*>(sm);
    Key* B = A + K;
    Key* H = B + K;
    Key* L = H + K;
    for (int i = threadIdx.x; i < 2 * K; i += T) A[i] = in[i];
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if constexpr (V == 0) {
            cta_merge_full<Key, K, T>(A, B, H, L);
        } else if constexpr (V == 1) {
            cta_merge_lo<Key, K, T>(A, B, H);  // first K only
        } else if constexpr (V == 2) {
            cta_merge_full2<Key, K, T>(A, B, H, L);
        } else if constexpr (V == 3) {
            cta_merge_tiles<Key, K, T, false, false>(A, B, H, L);
        } else if constexpr (V == 4) {
            cta_merge_first<Key, K, T, false>(A, B, H);
        } else if constexpr (V == 6) {
            cta_merge_q<Key, K, T, false, false>(A, B, H, L);
        } else if constexpr (V == 7) {
            cta_merge_q_first<Key, K, T, false>(A, B, H);
        } else if constexpr (V == 8) {
            cta_merge_qv<Key, K, T, false, false>(A, B, H, L);
        }  // V == 5: empty
        __syncthreads();
        // feed outputs back so the compiler cannot hoist anything
        if (threadIdx.x == 0) A[0] = H[0] < A[0] ? H[0] : A[0];
        __syncthreads();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
    for (int i = threadIdx.x; i < K; i += T) sink[i] = H[i] ^ L[i];
}

template <typename Key, int K, int T, int V>
__global__ void __launch_bounds__(T) merge_once(const Key* in, Key* out) {
    extern __shared__ __align__(16) unsigned char sm[];
    Key* A = reinterpret_cast<Key*>(sm);
    Key* B = A + K;
    Key* H = B + K;
    Key* L = H + K;
    for (int i = threadIdx.x; i < 2 * K; i += T) A[i] = in[i];
    for (int i = threadIdx.x; i < 2 * K; i += T) H[i] = 0;
    __syncthreads();
    if constexpr (V == 0) cta_merge_full<Key, K, T>(A, B, H, L);
    else if constexpr (V == 1) cta_merge_lo<Key, K, T>(A, B, H);
    else if constexpr (V == 2) cta_merge_full2<Key, K, T>(A, B, H, L);
    else if constexpr (V == 3) cta_merge_tiles<Key, K, T, false, false>(A, B, H, L);
    else if constexpr (V == 4) cta_merge_first<Key, K, T, false>(A, B, H);
    else if constexpr (V == 6) cta_merge_q<Key, K, T, false, false>(A, B, H, L);
    else if constexpr (V == 7) cta_merge_q_first<Key, K, T, false>(A, B, H);
    else if constexpr (V == 8) cta_merge_qv<Key, K, T, false, false>(A, B, H, L);
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * K; i += T) out[i] = H[i];
}

template <typename Key, int K, int T, int V>
__global__ void __launch_bounds__(T) sort_bench(const Key* in, int iters, unsigned long long* out, Key* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    Key* A = reinterpret_cast<Key*>(sm);
    unsigned long long tot = 0;
    for (int it = 0; it < iters; ++it) {
        for (int i = threadIdx.x; i < K; i += T) A[i] = in[(i * 7 + it) % K];
        __syncthreads();
        unsigned long long t0 = clock64();
        if constexpr (V == 0) cta_bitonic_sort<Key, K, T>(A);
        else if constexpr (V == 1) cta_sort_regs<Key, K, T>(A);
        else cta_sort_merge<Key, K, T>(A, A + K);
        unsigned long long t1 = clock64();
        tot += t1 - t0;
        for (int i = threadIdx.x; i + 1 < K; i += T)
            if (A[i] > A[i + 1]) sink[K] = 1;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = tot / iters;
    for (int i = threadIdx.x; i < K; i += T) sink[i] = A[i];
}

// Two CTAs (block 0 and block `other`) pass a node back and forth.
// MODE bits: 1 = load the node after the claim, 2 = store it before the
// release, 4 = relaxed polls + one fence (instead of ld.acquire polls),
// 8 = CAS claim (else a plain relaxed store of INUSE).
template <int K, int T, int MODE>
__global__ void __launch_bounds__(T) handoff_bench(uint32_t* node, uint32_t* st, int iters, int other,
                                                   unsigned long long* out) {
    __shared__ __align__(16) uint32_t buf[K];
    __shared__ uint32_t w_sh;
    int me;
    if (blockIdx.x == 0) me = 0;
    else if ((int)blockIdx.x == other) me = 1;
    else return;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) {
            uint32_t w;
            for (;;) {
                if constexpr (MODE & 4) {
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(w) : "l"(st) : "memory");
                } else {
                    w = state_load(st);
                }
                if (((w >> 3) & 1u) == (uint32_t)me) break;
            }
            if constexpr (MODE & 4) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            w_sh = w;
        }
        __syncthreads();
        if constexpr (MODE & 1) cta_load<uint32_t, T>(buf, node, K);
        if (threadIdx.x == 0) {
            uint32_t w = w_sh;
            if constexpr (MODE & 8) state_cas(st, w, swith(w, kInUse));
            else asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(st), "r"(swith(w, kInUse)) : "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) buf[0] += 1;
        __syncthreads();
        if constexpr (MODE & 2) cta_store<uint32_t, T>(node, buf, K);
        __syncthreads();
        if (threadIdx.x == 0) state_release(st, kInUse, kAvail);
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[me] = (t1 - t0) / iters;
}

// Latency of loading one 4 KiB node (just written by another SM) into
// shared memory: VEC bytes per thread (4, 8, 16), NT threads issuing.
template <int VEC, int NT>
__global__ void __launch_bounds__(512) nodeload_bench(uint32_t* node, uint32_t* flag, int iters, int other,
                                                     unsigned long long* out) {
    __shared__ __align__(16) uint32_t buf[1024];
    int me;
    if (blockIdx.x == 0) me = 0;
    else if ((int)blockIdx.x == other) me = 1;
    else return;
    unsigned long long tot = 0;
    for (int it = 0; it < iters; ++it) {
        if (me == 1) {
            // writer: rewrite the node, publish
            for (int i = threadIdx.x; i < 256; i += 512) __stcg(reinterpret_cast<uint4*>(node) + i, make_uint4(it, it, it, it));
            __syncthreads();
            if (threadIdx.x == 0) { __threadfence(); atomicExch(flag, (uint32_t)(2 * it + 1)); }
            if (threadIdx.x == 0) while (state_load(flag) != (uint32_t)(2 * it + 2)) {}
            __syncthreads();
        } else {
            if (threadIdx.x == 0) while (state_load(flag) != (uint32_t)(2 * it + 1)) {}
            __syncthreads();
            unsigned long long t0 = clock64();
            if (threadIdx.x < NT) {
                if constexpr (VEC == 16) {
                    for (int i = threadIdx.x; i < 256; i += NT) reinterpret_cast<uint4*>(buf)[i] = __ldcg(reinterpret_cast<const uint4*>(node) + i);
                } else if constexpr (VEC == 8) {
                    for (int i = threadIdx.x; i < 512; i += NT) reinterpret_cast<uint2*>(buf)[i] = __ldcg(reinterpret_cast<const uint2*>(node) + i);
                } else {
                    for (int i = threadIdx.x; i < 1024; i += NT) buf[i] = __ldcg(node + i);
                }
            }
            __syncthreads();
            unsigned long long t1 = clock64();
            tot += t1 - t0;
            if (threadIdx.x == 0) { if (buf[5] != (uint32_t)it) tot += 1000000000ull; atomicExch(flag, (uint32_t)(2 * it + 2)); }
            __syncthreads();
        }
    }
    if (me == 0 && threadIdx.x == 0) out[0] = tot / iters;
}

template <int VEC, int NT>
void run_nodeload(const char* name) {
    uint32_t *node, *flag;
    unsigned long long* o;
    CK(cudaMalloc(&node, 4096));
    CK(cudaMalloc(&flag, 256));
    CK(cudaMemset(flag, 0, 256));
    CK(cudaMalloc(&o, 16));
    nodeload_bench<VEC, NT><<<148, 512>>>(node, flag, 2000, 74, o);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("nodeload %-12s vec=%2d threads=%3d : %llu cycles\n", name, VEC, NT, c);
    cudaFree(node); cudaFree(flag); cudaFree(o);
}

// Round trip of one atomicCAS / red+poll from a single thread.
__global__ void atom_rt(uint32_t* p, int iters, unsigned long long* out) {
    unsigned long long t0 = clock64();
    uint32_t v = 0;
    for (int i = 0; i < iters; ++i) v = atomicCAS(p, v, v + 1);
    unsigned long long t1 = clock64();
    out[0] = (t1 - t0) / iters;
    out[1] = v;
}

// Basic latencies inside one CTA of T threads: dependent LDS chain, dependent
// SHFL chain, bar.sync, and an empty loop.
template <int T, int WHAT>
__global__ void __launch_bounds__(T) lat_bench(int iters, unsigned long long* out, unsigned* sink) {
    __shared__ unsigned s[1024];
    for (int i = threadIdx.x; i < 1024; i += T) s[i] = (i * 37 + 11) & 1023;
    __syncthreads();
    unsigned x = threadIdx.x & 1023;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if constexpr (WHAT == 0) x = s[x];                                   // LDS chain
        else if constexpr (WHAT == 1) x = __shfl_xor_sync(0xFFFFFFFFu, x, 1) + 1;  // SHFL chain
        else if constexpr (WHAT == 2) { __syncthreads(); x += 1; }            // barrier
        else if constexpr (WHAT == 3) { x = x * 3 + 1; }                      // ALU
        else if constexpr (WHAT == 4) { x = __ballot_sync(0xFFFFFFFFu, x & 1) + x; }  // vote
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    sink[threadIdx.x] = x;
}

template <int T, int WHAT>
void run_lat(const char* name) {
    unsigned long long* o;
    unsigned* sink;
    CK(cudaMalloc(&o, 16));
    CK(cudaMalloc(&sink, 4 * 1024));
    lat_bench<T, WHAT><<<1, T>>>(10000, o, sink);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("lat %-10s T=%4d : %llu cycles\n", name, T, c);
    cudaFree(o); cudaFree(sink);
}

__global__ void chase(const unsigned* p, int iters, unsigned long long* out) {
    unsigned idx = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) idx = __ldcg(p + idx);
    unsigned long long t1 = clock64();
    out[0] = (t1 - t0) / iters;
    out[1] = idx;
}

template <int K, int T, int V>
void run_merge(const char* name) {
    using Key = uint32_t;
    std::mt19937 rng(1);
    std::vector<Key> h(2 * K);
    for (auto& x : h) x = rng() >> 1;
    std::sort(h.begin(), h.begin() + K);
    std::sort(h.begin() + K, h.end());
    Key *d, *sink;
    unsigned long long* o;
    CK(cudaMalloc(&d, 2 * K * 4));
    CK(cudaMalloc(&sink, 2 * K * 4 + 16));
    CK(cudaMalloc(&o, 8 * 8));
    CK(cudaMemcpy(d, h.data(), 2 * K * 4, cudaMemcpyHostToDevice));
    auto kern = merge_bench<Key, K, T, V>;
    const int smem = 4 * K * 4 + 64;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, T, smem>>>(d, 2000, o, sink);
    CK(cudaDeviceSynchronize());
    {
        auto k1 = merge_once<Key, K, T, V>;
        CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k1<<<1, T, smem>>>(d, sink);
        CK(cudaDeviceSynchronize());
        std::vector<Key> got(2 * K), ref(2 * K);
        CK(cudaMemcpy(got.data(), sink, 2 * K * 4, cudaMemcpyDeviceToHost));
        std::merge(h.begin(), h.begin() + K, h.begin() + K, h.end(), ref.begin());
        const int n = V == 5 ? 0 : (V == 1 || V == 4 || V == 7) ? K : 2 * K;
        if (!std::equal(ref.begin(), ref.begin() + n, got.begin())) printf("merge %s: WRONG OUTPUT\n", name);
    }
    unsigned long long c;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    printf("merge %-22s K=%d T=%d : %llu cycles\n", name, K, T, c);
    cudaFree(d); cudaFree(sink); cudaFree(o);
}

template <int K, int T, int V>
void run_sort(const char* name) {
    using Key = uint32_t;
    std::mt19937 rng(2);
    std::vector<Key> h(K);
    for (auto& x : h) x = rng() >> 1;
    Key *d, *sink;
    unsigned long long* o;
    CK(cudaMalloc(&d, K * 4));
    CK(cudaMalloc(&sink, 2 * K * 4 + 16));
    CK(cudaMemset(sink, 0, 2 * K * 4 + 16));
    CK(cudaMalloc(&o, 8 * 8));
    CK(cudaMemcpy(d, h.data(), K * 4, cudaMemcpyHostToDevice));
    auto kern = sort_bench<Key, K, T, V>;
    sort_bench<Key, K, T, V><<<1, T, 2 * K * 4>>>(d, 200, o, sink);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    Key bad;
    CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&bad, sink + K, 4, cudaMemcpyDeviceToHost));
    std::vector<Key> res(K);
    CK(cudaMemcpy(res.data(), sink, K * 4, cudaMemcpyDeviceToHost));
    printf("sort  %-22s K=%d T=%d : %llu cycles %s\n", name, K, T, c, bad ? "UNSORTED" : "ok");
    cudaFree(d); cudaFree(sink); cudaFree(o);
    (void)kern;
}

template <int MODE>
void run_handoff(int other, const char* name) {
    static bool once = false;
    if (!once) {
        once = true;
        uint32_t* p;
        unsigned long long* o;
        CK(cudaMalloc(&p, 256));
        CK(cudaMemset(p, 0, 256));
        CK(cudaMalloc(&o, 16));
        atom_rt<<<1, 1>>>(p, 10000, o);
        CK(cudaDeviceSynchronize());
        unsigned long long c[2];
        CK(cudaMemcpy(c, o, 16, cudaMemcpyDeviceToHost));
        printf("atomicCAS round trip (dependent): %llu cycles\n", c[0]);
        cudaFree(p); cudaFree(o);
    }
    uint32_t *node, *st;
    unsigned long long* o;
    CK(cudaMalloc(&node, 4096));
    CK(cudaMalloc(&st, 256));
    CK(cudaMemset(st, 0, 256));
    CK(cudaMemset(node, 0, 4096));
    CK(cudaMalloc(&o, 16));
    handoff_bench<1024, 512, MODE><<<148, 512>>>(node, st, 4000, other, o);
    CK(cudaDeviceSynchronize());
    unsigned long long c[2];
    CK(cudaMemcpy(c, o, 16, cudaMemcpyDeviceToHost));
    printf("handoff %-20s other=%3d : %llu cycles per pass (half round trip)\n", name, other, c[0] / 2);
    cudaFree(node); cudaFree(st); cudaFree(o);
}

int main(int argc, char** argv) {
    if (argc > 1) {
        std::string w = argv[1];
        if (w == "pad") {
            run_half<1024, 512, 4, 0>("binary");
            run_halfpad<1024, 512, 4>("padded binary");
            run_halfpad<1024, 512, 2>("padded binary");
            run_halfpad<1024, 512, 8>("padded binary");
            run_halfpad<1024, 256, 4>("padded binary");
        }
        if (w == "half") {
            run_half<1024, 512, 4, 0>("binary");
            run_half<1024, 512, 4, 1>("quaternary");
            run_half<1024, 512, 2, 0>("binary");
            run_half<1024, 512, 2, 1>("quaternary");
            run_half<1024, 512, 8, 0>("binary");
            run_half<1024, 512, 8, 1>("quaternary");
            run_half<1024, 512, 1, 1>("quaternary");
            run_half<1024, 256, 4, 1>("quaternary");
        }
        if (w == "bt") {
            run_halfbt<1024, 128, 8>("warp bitonic");
            run_halfbt<1024, 256, 4>("warp bitonic");
            run_halfbt<1024, 512, 2>("warp bitonic");
            run_halfbt<1024, 256, 2>("warp bitonic 2 tiles");
            run_halfbt<1024, 512, 1>("warp bitonic 2 tiles");
            run_halfbt<2048, 512, 4>("warp bitonic");
            run_halfbt<2048, 256, 8>("warp bitonic");
            run_halfbt<256, 64, 4>("warp bitonic");
            run_halfbt<256, 128, 2>("warp bitonic");
            run_half<1024, 256, 4, 0>("binary");
            run_half<1024, 512, 2, 0>("binary");
        }
        if (w == "groups") {  // half merge on one thread group of T threads (P outputs each)
            run_half<1024, 128, 8, 0>("binary");
            run_half<1024, 256, 4, 0>("binary");
            run_half<1024, 512, 2, 0>("binary");
            run_half<1024, 1024, 1, 0>("binary");
            run_half<1024, 128, 8, 1>("quaternary");
            run_half<1024, 256, 4, 1>("quaternary");
            run_half<256, 64, 4, 0>("binary");
            run_half<256, 32, 8, 0>("binary");
            run_half<2048, 256, 8, 0>("binary");
            run_half<2048, 512, 4, 0>("binary");
            run_lat<128, 2>("bar");
            run_lat<256, 2>("bar");
        }
        if (w == "load") {
            run_nodeload<16, 256>("remote-written");
            run_nodeload<16, 512>("remote-written");
            run_nodeload<16, 128>("remote-written");
            run_nodeload<8, 512>("remote-written");
            run_nodeload<4, 512>("remote-written");
            run_handoff<1 | 2 | 8>(74, "full (ld.acq polls)");
            run_handoff<2 | 8>(74, "store only");
            run_handoff<1 | 8>(74, "load only");
            run_handoff<8>(74, "state only, CAS");
            run_handoff<0>(74, "state only, store");
        }
        if (w == "m0") run_merge<1024, 512, 0>("full (current)");
        if (w == "m8") run_merge<1024, 512, 8>("quaternary E8 vec full");
        if (w == "m3") run_merge<1024, 512, 3>("warp tiles full");
        if (w == "s0") run_sort<1024, 512, 0>("bitonic smem");
        if (w == "s2") run_sort<1024, 512, 2>("merge passes");
        return 0;
    }
    {
        unsigned* p;
        unsigned long long* o;
        const int n = 1 << 22;
        std::vector<unsigned> h(n);
        std::mt19937 rng(3);
        // random cycle within the first 64 KiB (L2-resident after the first pass)
        const int m = 16384;
        std::vector<unsigned> perm(m);
        for (int i = 0; i < m; ++i) perm[i] = i;
        std::shuffle(perm.begin() + 1, perm.end(), rng);
        for (int i = 0; i < m; ++i) h[perm[i] * 1] = perm[(i + 1) % m];
        CK(cudaMalloc(&p, n * 4));
        CK(cudaMalloc(&o, 16));
        CK(cudaMemcpy(p, h.data(), n * 4, cudaMemcpyHostToDevice));
        chase<<<1, 1>>>(p, 20000, o);
        CK(cudaDeviceSynchronize());
        unsigned long long c[2];
        CK(cudaMemcpy(c, o, 16, cudaMemcpyDeviceToHost));
        printf("L2 pointer chase: %llu cycles per dependent ld.cg\n", c[0]);
    }
    run_lat<32, 0>("lds");
    run_lat<512, 0>("lds");
    run_lat<32, 1>("shfl");
    run_lat<512, 1>("shfl");
    run_lat<32, 2>("bar");
    run_lat<512, 2>("bar");
    run_lat<32, 3>("alu");
    run_lat<32, 4>("ballot");
    run_merge<1024, 512, 5>("empty loop");
    run_merge<1024, 512, 0>("full (current)");
    run_merge<1024, 512, 1>("first-K only");
    run_merge<1024, 512, 2>("full v2");
    run_merge<1024, 512, 8>("quaternary E8 vec full");
    run_merge<2048, 512, 8>("quaternary E8 vec full");
    run_merge<256, 128, 8>("quaternary E8 vec full");
    run_merge<1024, 512, 6>("quaternary E8 full");
    run_merge<1024, 512, 7>("quaternary E8 first-K");
    run_merge<2048, 512, 6>("quaternary full");
    run_merge<256, 128, 6>("quaternary full");
    run_merge<64, 32, 6>("quaternary full");
    run_merge<16, 32, 6>("quaternary full");
    run_merge<1024, 512, 3>("warp tiles full");
    run_merge<1024, 512, 4>("warp tiles first-K");
    run_merge<2048, 512, 0>("full (current)");
    run_merge<2048, 512, 3>("warp tiles full");
    run_merge<256, 128, 3>("warp tiles full");
    run_merge<64, 32, 3>("warp tiles full");
    run_merge<16, 32, 3>("warp tiles full");
    run_merge<1024, 256, 0>("full (current)");
    run_merge<1024, 256, 2>("full v2");
    run_merge<256, 128, 0>("full (current)");
    run_merge<256, 128, 2>("full v2");
    run_sort<1024, 512, 0>("bitonic smem");
    run_sort<1024, 512, 1>("bitonic regs");
    run_sort<1024, 512, 2>("merge passes");
    run_sort<2048, 512, 0>("bitonic smem");
    run_sort<2048, 512, 2>("merge passes");
    run_sort<256, 128, 2>("merge passes");
    run_sort<64, 32, 2>("merge passes");
    run_sort<256, 128, 0>("bitonic smem");
    run_sort<256, 128, 1>("bitonic regs");
    for (int other : {1, 74, 147}) run_handoff<1 | 2 | 8>(other, "full (ld.acq polls)");
    run_handoff<1 | 2 | 8 | 4>(74, "full (relaxed polls)");
    run_handoff<8>(74, "state only, CAS");
    run_handoff<0>(74, "state only, store");
    run_handoff<4>(74, "state only, relaxed");
    run_handoff<1 | 8>(74, "load only");
    run_handoff<2 | 8>(74, "store only");
    return 0;
}

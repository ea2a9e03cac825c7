// bh_select.cuh -- latency-tuned CTA merge building blocks of the heap.
//
// The heap's throughput is a chain of dependent per-level steps (claim,
// merge, write back, release), so these primitives are tuned for the
// latency of one CTA:
//   * merge-path splits use a fixed-trip branchless search (no divergence);
//   * each thread preloads its whole A/B window (independent LDS, one
//     latency) and merges it in registers with selects;
//   * a level needs the two halves of a merge at different times, so the
//     merge is split into half merges (outputs [0,K) or [K,2K)).
// Variants measured and rejected (warp-tile bitonic, quaternary search,
// vector windows, padded layouts, register sorts) live with their
// microbenchmark in tools/microbench/mb_variants.cuh.
#pragma once

#include "bh_device.cuh"

namespace bh {

// Largest i in [lo, hi] with (i == lo || A[i-1] <= B[d-i]): the number of A
// elements among the first d outputs of the stable (A-first) merge.
template <typename Key, int K>
__device__ __forceinline__ uint32_t merge_split(const Key* __restrict__ A, const Key* __restrict__ B,
                                                uint32_t d, uint32_t na, uint32_t nb) {
    const uint32_t lo = d > nb ? d - nb : 0;
    const uint32_t hi = d < na ? d : na;
    uint32_t base = lo;
#pragma unroll
    for (uint32_t step = (uint32_t)K; step > 0; step >>= 1) {
        const uint32_t p = base + step;
        if (p <= hi && A[p - 1] <= B[d - p]) base = p;
    }
    return base;
}

// Merges the window A[i..), B[j..) in registers: the next N outputs of the
// stable merge, given the remaining lengths.  Sentinel-padded loads keep the
// network branch-free (ties take A, and a real A key equal to the pad never
// loses to it because the pad is only taken once A is exhausted).
template <typename Key, int N>
__device__ __forceinline__ void merge_window(const Key* __restrict__ A, uint32_t i, uint32_t na,
                                             const Key* __restrict__ B, uint32_t j, uint32_t nb,
                                             Key (&out)[N]) {
    Key a[N + 1], b[N + 1];
#pragma unroll
    for (int e = 0; e < N; ++e) {
        a[e] = i + e < na ? A[i + e] : KeyLimits<Key>::kMax;
        b[e] = j + e < nb ? B[j + e] : KeyLimits<Key>::kMax;
    }
    a[N] = KeyLimits<Key>::kMax;
    b[N] = KeyLimits<Key>::kMax;
    // remaining counts decide ties with the pad: A exhausted => take B
    uint32_t ra = na - i, rb = nb - j;
#pragma unroll
    for (int e = 0; e < N; ++e) {
        const bool take_a = rb == 0 || (ra != 0 && a[0] <= b[0]);
        out[e] = take_a ? a[0] : b[0];
#pragma unroll
        for (int s = 0; s < N; ++s) {
            a[s] = take_a ? a[s + 1] : a[s];
            b[s] = take_a ? b[s] : b[s + 1];
        }
        ra -= take_a;
        rb -= !take_a;
    }
}

template <typename Key, int N>
__device__ __forceinline__ void store_run(Key* dst, const Key (&run)[N]) {
    constexpr uint32_t kBytes = N * sizeof(Key);
    if constexpr (kBytes % 16 == 0) {
        if (((uint32_t)(uintptr_t)dst & 15u) == 0) {
            uint4* dv = reinterpret_cast<uint4*>(dst);
            const uint4* rv = reinterpret_cast<const uint4*>(run);
#pragma unroll
            for (uint32_t v = 0; v < kBytes / 16; ++v) dv[v] = rv[v];
            return;
        }
    }
#pragma unroll
    for (int e = 0; e < N; ++e) dst[e] = run[e];
}

// Global stores through L2 (the heap's node arrays).
template <typename Key, int N>
__device__ __forceinline__ void store_run_cg(Key* dst, const Key (&run)[N]) {
    constexpr uint32_t kBytes = N * sizeof(Key);
    if constexpr (kBytes % 16 == 0) {
        uint4* dv = reinterpret_cast<uint4*>(dst);
        const uint4* rv = reinterpret_cast<const uint4*>(run);
#pragma unroll
        for (uint32_t v = 0; v < kBytes / 16; ++v) __stcg(dv + v, rv[v]);
    } else {
#pragma unroll
        for (int e = 0; e < N; ++e) __stcg(dst + e, run[e]);
    }
}

// One half of merge_and_sort(A, B) on two full K-batches: outputs [0, K)
// (the hi batch) when !Second, [K, 2K) (the lo batch) when Second, written
// to `out` (through L2 when Global).  A heapify level releases its node
// after the first halves and finishes the second halves afterwards.  `tid`
// is the calling thread's index within the group doing this merge
// (HalfShape::kThreads threads; others return).  No barrier inside.
template <int K, int T>
struct HalfShape {
    static constexpr int P0 = (K + T - 1) / T;
    static constexpr int P = (K >= 4 && K / 4 <= T) ? 4 : (P0 < 1 ? 1 : P0);
    static constexpr int kThreads = K / P;
    // two halves can run side by side on disjoint thread groups
    static constexpr bool kPair = 2 * kThreads <= T;
};

template <typename Key, int K, int T, bool Second, bool Global>
__device__ __forceinline__ void cta_merge_half(const Key* __restrict__ A, const Key* __restrict__ B,
                                               Key* __restrict__ out, uint32_t tid, uint32_t nthr) {
    constexpr int P = HalfShape<K, T>::P;
    for (uint32_t t0 = tid * P; t0 < (uint32_t)K; t0 += nthr * P) {
        const uint32_t d0 = (Second ? (uint32_t)K : 0u) + t0;
        const uint32_t i = merge_split<Key, K>(A, B, d0, K, K);
        Key run[P];
        merge_window<Key, P>(A, i, K, B, d0 - i, K, run);
        if constexpr (Global) store_run_cg<Key, P>(out + t0, run);
        else store_run<Key, P>(out + t0, run);
    }
}

// cta_merge_half with an explicit window P (K / P threads cover a half);
// the delete server runs both halves of a sibling merge side by side on one
// thread group with it.
template <typename Key, int K, int P, bool Second, bool Global>
__device__ __forceinline__ void cta_merge_half_p(const Key* __restrict__ A, const Key* __restrict__ B,
                                                 Key* __restrict__ out, uint32_t tid, uint32_t nthr) {
    for (uint32_t t0 = tid * P; t0 < (uint32_t)K; t0 += nthr * P) {
        const uint32_t d0 = (Second ? (uint32_t)K : 0u) + t0;
        const uint32_t i = merge_split<Key, K>(A, B, d0, K, K);
        Key run[P];
        merge_window<Key, P>(A, i, K, B, d0 - i, K, run);
        if constexpr (Global) store_run_cg<Key, P>(out + t0, run);
        else store_run<Key, P>(out + t0, run);
    }
}

}  // namespace bh

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
// The half merges of the heap use the warp-tile bitonic merge at the end of
// this file (warp_half_bt); the per-thread merge path above remains for
// unequal lengths and K < 32.  Variants measured and rejected (quaternary
// search, vector windows, padded layouts, register sorts) live with their
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

// ------------------------------------------------ warp-tile bitonic half --
// One half of merge_and_sort(A, B) on two sorted K-batches, by the NW warps
// of a thread group (`gw` = the calling warp's index within the group; all 32
// lanes of each warp call).  Each warp owns a tile of 32E consecutive
// outputs [D, D + 32E):
//   1. the merge-path split of diagonal D (how many A keys precede output D)
//      by a fixed-trip 32-ary search: lane l tests lo + (l+1)g for an odd
//      stride g (32 probes never share a bank), ballot + popc, the range
//      shrinks 32x per round (two rounds up to K = 1024);
//   2. the tile is the 32E smallest keys of the windows A[a, a+32E) and
//      B[b, b+32E) (sentinel past the ends), and min(Aw[i], Bw[32E-1-i]) is
//      a bitonic sequence holding exactly them;
//   3. a bitonic half-cleaner network sorts it: strides >= 32 inside each
//      lane's registers, strides < 32 with warp shuffles.  Lane l ends with
//      outputs D + 32e + l (coalesced stores).
// Keys carry no payload, so the output equals the reference's stable
// merge_sorted (proj/src/batch.cpp:21-42) key for key.  Measured (tools/
// microbench `mb bt`, K=1024, 4 warps): 695 cycles per half vs 1954 for the
// per-thread merge path on the same 128 threads (1089 on 256).
// Not inlined: inlined into heap_ops_kernel (CUDA 12.9 ptxas, sm_100a) the
// second-half tiles computed by warps 0-2 in heapify's phase 2 came out wrong
// for correct, stable inputs -- deterministically, and again when recomputed
// after a barrier -- while the same inputs replayed standalone
// (tools/microbench/bt_check <dump>) and the out-of-line function are right.
template <typename Key, int K, int E, bool Global>
__device__ __noinline__ void warp_half_bt(const Key* __restrict__ A, const Key* __restrict__ B,
                                             Key* __restrict__ out, uint32_t D) {
    constexpr uint32_t W = 32u * E;
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t lo = D > (uint32_t)K ? D - K : 0u;
    uint32_t hi = D < (uint32_t)K ? D : (uint32_t)K;
#pragma unroll
    for (uint32_t span = (uint32_t)K; span > 0; span >>= 5) {
        const uint32_t g = span > 32 ? ((span + 31u) >> 5) | 1u : 1u;
        const uint32_t p = lo + (lane + 1u) * g;
        const bool ok = p <= hi && A[p - 1] <= B[D - p];
        lo += (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, ok)) * g;
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
        const bool upper = (lane & (uint32_t)ls) != 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const Key o = __shfl_xor_sync(0xFFFFFFFFu, v[e], ls);
            v[e] = upper ? (v[e] < o ? o : v[e]) : (v[e] < o ? v[e] : o);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if constexpr (Global) __stcg(out + e * 32u + lane, v[e]);
        else out[e * 32u + lane] = v[e];
    }
}

// The same network inlined (no call: the caller's live registers are not
// saved to the stack around it), for the three-level delete server's merges.
template <typename Key, int K, int E, bool Global>
__device__ __forceinline__ void warp_half_bt_inl(const Key* __restrict__ A, const Key* __restrict__ B,
                                             Key* __restrict__ out, uint32_t D) {
    constexpr uint32_t W = 32u * E;
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t lo = D > (uint32_t)K ? D - K : 0u;
    uint32_t hi = D < (uint32_t)K ? D : (uint32_t)K;
#pragma unroll
    for (uint32_t span = (uint32_t)K; span > 0; span >>= 5) {
        const uint32_t g = span > 32 ? ((span + 31u) >> 5) | 1u : 1u;
        const uint32_t p = lo + (lane + 1u) * g;
        const bool ok = p <= hi && A[p - 1] <= B[D - p];
        lo += (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, ok)) * g;
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
        const bool upper = (lane & (uint32_t)ls) != 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const Key o = __shfl_xor_sync(0xFFFFFFFFu, v[e], ls);
            v[e] = upper ? (v[e] < o ? o : v[e]) : (v[e] < o ? v[e] : o);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if constexpr (Global) __stcg(out + e * 32u + lane, v[e]);
        else out[e * 32u + lane] = v[e];
    }
}

// The inlined network with the output space chosen at run time.  Every
// shared-memory load is unconditional, at a clamped index, with the bound
// applied by a select afterwards: predicated loads into one temporary would
// serialise the window (each load waits for the previous one's move), which
// under the register pressure of the server's loop costs more than the
// merge itself.
template <typename Key, int K, int E>
__device__ __forceinline__ void warp_half_bt_rt(const Key* __restrict__ A, const Key* __restrict__ B,
                                                Key* __restrict__ out, uint32_t D, bool global) {
    constexpr uint32_t W = 32u * E;
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t lo = D > (uint32_t)K ? D - K : 0u;
    uint32_t hi = D < (uint32_t)K ? D : (uint32_t)K;
#pragma unroll
    for (uint32_t span = (uint32_t)K; span > 0; span >>= 5) {
        const uint32_t g = span > 32 ? ((span + 31u) >> 5) | 1u : 1u;
        const uint32_t p = lo + (lane + 1u) * g;
        const uint32_t pc = p <= hi ? p : hi;  // hi >= 1 when lo < hi; else no lane is ok
        const uint32_t ia = pc ? pc - 1u : 0u;
        const uint32_t ib = D - pc < (uint32_t)K ? D - pc : (uint32_t)K - 1u;
        const Key xa = A[ia], xb = B[ib];
        const bool ok = p <= hi && xa <= xb;
        lo += (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, ok)) * g;
        const uint32_t h2 = lo + g - 1u;
        hi = h2 < hi ? h2 : hi;
        if (g == 1u) break;
    }
    const uint32_t a = lo, b = D - lo;
    Key v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const uint32_t i = e * 32u + lane;
        const bool ina = a + i < (uint32_t)K;
        const Key x0 = A[ina ? a + i : (uint32_t)K - 1u];
        const uint32_t j = b + (W - 1u - i);
        const bool inb = j < (uint32_t)K;
        const Key y0 = B[inb ? j : (uint32_t)K - 1u];
        const Key x = ina ? x0 : KeyLimits<Key>::kMax;
        const Key y = inb ? y0 : KeyLimits<Key>::kMax;
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
        const bool upper = (lane & (uint32_t)ls) != 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const Key o = __shfl_xor_sync(0xFFFFFFFFu, v[e], ls);
            v[e] = upper ? (v[e] < o ? o : v[e]) : (v[e] < o ? v[e] : o);
        }
    }
    if (global) {
#pragma unroll
        for (int e = 0; e < E; ++e) __stcg(out + e * 32u + lane, v[e]);
    } else {
#pragma unroll
        for (int e = 0; e < E; ++e) out[e * 32u + lane] = v[e];
    }
}

// Tile shape of a half merge on NW warps: each used warp covers kPer outputs
// in tiles of 32E (E <= 16 keys per lane).
template <int K, int NW>
struct TileShape {
    static constexpr int kUsed = K >= 32 * NW ? NW : (K >= 32 ? K / 32 : 0);  // 0: K < 32
    static constexpr int kPer = kUsed ? K / kUsed : 0;
    static constexpr int E = kPer / 32 > 16 ? 16 : kPer / 32;
    static constexpr int kTiles = E ? kPer / (32 * E) : 0;
};

// Outputs [0, K) (!Second) or [K, 2K) (Second) of merge(A, B) -> out[0, K),
// by the NW warps of a group (gw = warp index in the group).  K < 32 falls
// back to the per-thread merge path on the group's threads.  No barrier.
template <typename Key, int K, int NW, bool Second, bool Global, bool Inl = false>
__device__ __forceinline__ void grp_merge_half(const Key* __restrict__ A, const Key* __restrict__ B,
                                               Key* __restrict__ out, uint32_t gw) {
    using S = TileShape<K, NW>;
    if constexpr (S::kUsed == 0) {
        cta_merge_half<Key, K, 32 * NW, Second, Global>(A, B, out, gw * 32u + (threadIdx.x & 31u), 32u * NW);
    } else {
        if (gw >= (uint32_t)S::kUsed) return;
#pragma unroll 1
        for (int t = 0; t < S::kTiles; ++t) {
            const uint32_t o = gw * (uint32_t)S::kPer + (uint32_t)t * 32u * S::E;
            if constexpr (Inl)
                warp_half_bt_inl<Key, K, S::E, Global>(A, B, out + o, (Second ? (uint32_t)K : 0u) + o);
            else
                warp_half_bt<Key, K, S::E, Global>(A, B, out + o, (Second ? (uint32_t)K : 0u) + o);
        }
    }
}

// The k-th smallest key (k = K) of two sorted K-batches -- the largest key
// of the first half of their merge -- by one warp (every lane gets it): the
// 32-ary merge-path split of diagonal K, then max(A[a-1], B[K-a-1]).
template <typename Key, int K>
__device__ __forceinline__ Key warp_kth_max(const Key* __restrict__ A, const Key* __restrict__ B) {
    const uint32_t lane = threadIdx.x & 31u;
    constexpr uint32_t D = (uint32_t)K;
    uint32_t lo = 0, hi = D;
#pragma unroll
    for (uint32_t span = (uint32_t)K; span > 0; span >>= 5) {
        const uint32_t g = span > 32 ? ((span + 31u) >> 5) | 1u : 1u;
        const uint32_t p = lo + (lane + 1u) * g;
        const bool ok = p <= hi && A[p - 1] <= B[D - p];
        lo += (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, ok)) * g;
        const uint32_t h2 = lo + g - 1u;
        hi = h2 < hi ? h2 : hi;
        if (g == 1u) break;
    }
    const uint32_t a = lo;
    const Key x = a > 0 ? A[a - 1] : Key(0);
    const Key y = a < D ? B[D - 1 - a] : Key(0);
    return x > y ? x : y;
}

// grp_merge_half with the half and the output space chosen at run time, on
// the inlined network: one call site serves every merge of a round loop.
template <typename Key, int K, int NW>
__device__ __forceinline__ void grp_merge_half_rt(const Key* __restrict__ A, const Key* __restrict__ B,
                                                  Key* __restrict__ out, uint32_t gw, bool second, bool global) {
    using S = TileShape<K, NW>;
    static_assert(S::kUsed == NW, "one tile row per warp");
#pragma unroll 1
    for (int t = 0; t < S::kTiles; ++t) {
        const uint32_t o = gw * (uint32_t)S::kPer + (uint32_t)t * 32u * S::E;
        warp_half_bt_rt<Key, K, S::E>(A, B, out + o, (second ? (uint32_t)K : 0u) + o, global);
    }
}

// merge_and_sort of two full K-batches on T threads: the first half on warps
// [0, T/64), the second on the rest (side by side).  No barrier.
template <typename Key, int K, int T, bool HiGlobal = false, bool LoGlobal = false>
__device__ __forceinline__ void cta_merge_full_bt(const Key* __restrict__ A, const Key* __restrict__ B,
                                                  Key* __restrict__ out_hi, Key* __restrict__ out_lo) {
    constexpr int kW = T / 32;
    if constexpr (kW >= 2) {
        constexpr int kH = kW / 2;
        const uint32_t w = threadIdx.x >> 5;
        if (w < (uint32_t)kH) grp_merge_half<Key, K, kH, false, HiGlobal>(A, B, out_hi, w);
        else if (w < 2u * kH) grp_merge_half<Key, K, kH, true, LoGlobal>(A, B, out_lo, w - kH);
    } else {
        grp_merge_half<Key, K, 1, false, HiGlobal>(A, B, out_hi, 0);
        grp_merge_half<Key, K, 1, true, LoGlobal>(A, B, out_lo, 0);
    }
}

}  // namespace bh

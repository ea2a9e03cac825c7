// mb_variants.cuh -- merge / sort variants measured by mb.cu against the
// product primitives (paper_1906_06504_b200/csrc/bh_select.cuh) and not
// adopted (tools/microbench results in DESIGN.md section 6).  Tooling only.
#pragma once

#include "../../paper_1906_06504_b200/csrc/bh_select.cuh"

namespace bh {

// Outputs per thread of a 2K merge on T threads (at least 1, at most 8 or
// whatever a 16-byte vector needs).
template <typename Key, int K, int T>
struct MergeShape {
    static constexpr int kVec = 16 / (int)sizeof(Key) < 1 ? 1 : 16 / (int)sizeof(Key);
    static constexpr int kRaw = (2 * K + T - 1) / T;
    static constexpr int kPer = kRaw < 1 ? 1 : kRaw;
    static constexpr int kThreads = (2 * K + kPer - 1) / kPer;  // active threads
};

// merge_and_sort of two full K-batches (proj/src/batch.cpp:32-42): the K
// smallest go to out_hi, the rest to out_lo (ties take A first).  Outputs are
// written with plain stores when `Global` is false (shared memory) and
// through L2 otherwise, per half.  No barrier inside.
template <typename Key, int K, int T, bool HiGlobal, bool LoGlobal>
__device__ __forceinline__ void cta_merge2(const Key* __restrict__ A, const Key* __restrict__ B,
                                           Key* __restrict__ out_hi, Key* __restrict__ out_lo) {
    using S = MergeShape<Key, K, T>;
    constexpr int P = S::kPer;
    const uint32_t d0 = threadIdx.x * P;
    if (d0 >= 2u * K) return;
    const uint32_t i = merge_split<Key, K>(A, B, d0, K, K);
    Key run[P];
    merge_window<Key, P>(A, i, K, B, d0 - i, K, run);
    if (d0 < (uint32_t)K) {
        if constexpr (HiGlobal) store_run_cg<Key, P>(out_hi + d0, run);
        else store_run<Key, P>(out_hi + d0, run);
    } else {
        if constexpr (LoGlobal) store_run_cg<Key, P>(out_lo + (d0 - K), run);
        else store_run<Key, P>(out_lo + (d0 - K), run);
    }
}

// First K outputs only (the hi half), into shared memory.
template <typename Key, int K, int T>
__device__ __forceinline__ void cta_merge_lo(const Key* __restrict__ A, const Key* __restrict__ B,
                                             Key* __restrict__ out_hi) {
    constexpr int P = (K + T - 1) / T < 4 ? ((K + T - 1) / T < 1 ? 1 : (K + T - 1) / T) : 4;
    const uint32_t d0 = threadIdx.x * P;
    if (d0 >= (uint32_t)K) return;
    const uint32_t i = merge_split<Key, K>(A, B, d0, K, K);
    Key run[P];
    merge_window<Key, P>(A, i, K, B, d0 - i, K, run);
    store_run<Key, P>(out_hi + d0, run);
}

template <typename Key, int K, int T>
__device__ __forceinline__ void cta_merge_full2(const Key* __restrict__ A, const Key* __restrict__ B,
                                                Key* __restrict__ out_hi, Key* __restrict__ out_lo) {
    cta_merge2<Key, K, T, false, false>(A, B, out_hi, out_lo);
}

// ------------------------------------------------------- warp-tile merge --
// Merge path split for two diagonals at once, found by the whole warp with a
// 32-ary search (2 rounds for spans up to 1024): lane l tests point
// lo + (l+1)*g, a ballot counts the true prefix of the monotone predicate
// P(i) = A[i-1] <= B[D-i], and the range shrinks 32x per round.  Returns the
// number of A elements among the first D0 (resp. D1) outputs of the stable
// (A-first) merge.  Warp-uniform; all 32 lanes must call it.
template <typename Key>
__device__ __forceinline__ void warp_split2(const Key* __restrict__ A, uint32_t na,
                                            const Key* __restrict__ B, uint32_t nb, uint32_t D0,
                                            uint32_t D1, uint32_t& s0, uint32_t& s1) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t lo0 = D0 > nb ? D0 - nb : 0, hi0 = D0 < na ? D0 : na;
    uint32_t lo1 = D1 > nb ? D1 - nb : 0, hi1 = D1 < na ? D1 : na;
    while (hi0 > lo0 || hi1 > lo1) {
        // odd strides: 32 probes g apart never share a shared-memory bank
        uint32_t g0 = (hi0 - lo0 + 31) >> 5, g1 = (hi1 - lo1 + 31) >> 5;
        g0 = g0 ? (g0 | 1u) : 0u;
        g1 = g1 ? (g1 | 1u) : 0u;
        const uint32_t i0 = lo0 + (lane + 1) * g0, i1 = lo1 + (lane + 1) * g1;
        const bool p0 = g0 != 0 && i0 <= hi0 && A[i0 - 1] <= B[D0 - i0];
        const bool p1 = g1 != 0 && i1 <= hi1 && A[i1 - 1] <= B[D1 - i1];
        const uint32_t c0 = __popc(__ballot_sync(0xFFFFFFFFu, p0));
        const uint32_t c1 = __popc(__ballot_sync(0xFFFFFFFFu, p1));
        lo0 += c0 * g0;
        hi0 = min(hi0, lo0 + (g0 ? g0 - 1 : 0));
        lo1 += c1 * g1;
        hi1 = min(hi1, lo1 + (g1 ? g1 - 1 : 0));
    }
    s0 = lo0;
    s1 = lo1;
}

// Outputs [D, D + 32E) of the stable merge of A[0,na) and B[0,nb), computed
// by one warp: the tile's A run (ascending) and B run (reversed) form a
// bitonic sequence of 32E keys in registers (position p = e*32 + lane), and a
// bitonic merge network sorts it -- in-register exchanges for strides >= 32,
// warp shuffles below.  Lane l ends with outputs D + e*32 + l.
template <typename Key, int E>
__device__ __forceinline__ void warp_merge_tile(const Key* __restrict__ A, uint32_t na,
                                                const Key* __restrict__ B, uint32_t nb, uint32_t D,
                                                Key (&v)[E]) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t a0, a1;
    warp_split2<Key>(A, na, B, nb, D, D + 32u * E, a0, a1);
    const uint32_t nA = a1 - a0;
    const uint32_t b1 = D + 32u * E - a1;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const uint32_t p = e * 32u + lane;
        v[e] = p < nA ? A[a0 + p] : B[b1 - 1 - (p - nA)];
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
            const Key mn = v[e] < o ? v[e] : o;
            const Key mx = v[e] < o ? o : v[e];
            v[e] = upper ? mx : mn;
        }
    }
}

template <typename Key, int E, bool Global>
__device__ __forceinline__ void warp_store_tile(Key* dst, const Key (&v)[E]) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if constexpr (Global) __stcg(dst + e * 32 + lane, v[e]);
        else dst[e * 32 + lane] = v[e];
    }
}

// Can the warp-tile merge cover a 2K (full) or K (first half) merge on T
// threads?  Each warp needs a power-of-two tile of >= 32 outputs.
template <int K, int T, bool Half>
struct WarpMerge {
    static constexpr int kWarps = T / 32;
    static constexpr int kOut = Half ? K : 2 * K;
    static constexpr int kTile = kWarps > 0 ? kOut / kWarps : 0;
    static constexpr int E = kTile / 32;
    static constexpr bool ok = kWarps > 0 && T % 32 == 0 && kTile >= 32 && kTile * kWarps == kOut &&
                               (kTile & (kTile - 1)) == 0 && (Half || kTile <= K) && E <= 16;
};

// merge_and_sort of two full K-batches (proj/src/batch.cpp:32-42) by warp
// tiles: outputs [0,K) -> hi, [K,2K) -> lo; each half to shared memory or
// through L2 to global memory.  No barrier inside.
template <typename Key, int K, int T, bool HiGlobal, bool LoGlobal>
__device__ __forceinline__ void cta_merge_tiles(const Key* __restrict__ A, const Key* __restrict__ B,
                                                Key* __restrict__ out_hi, Key* __restrict__ out_lo) {
    using W = WarpMerge<K, T, false>;
    if constexpr (W::ok) {
        const uint32_t D = (threadIdx.x >> 5) * W::kTile;
        Key v[W::E];
        warp_merge_tile<Key, W::E>(A, K, B, K, D, v);
        if (D < (uint32_t)K) warp_store_tile<Key, W::E, HiGlobal>(out_hi + D, v);
        else warp_store_tile<Key, W::E, LoGlobal>(out_lo + (D - K), v);
    } else {
        cta_merge_full<Key, K, T>(A, B, out_hi, out_lo);
    }
}

// The first K outputs only.
template <typename Key, int K, int T, bool HiGlobal>
__device__ __forceinline__ void cta_merge_first(const Key* __restrict__ A, const Key* __restrict__ B,
                                                Key* __restrict__ out_hi) {
    using W = WarpMerge<K, T, true>;
    if constexpr (W::ok) {
        const uint32_t D = (threadIdx.x >> 5) * W::kTile;
        Key v[W::E];
        warp_merge_tile<Key, W::E>(A, K, B, K, D, v);
        warp_store_tile<Key, W::E, HiGlobal>(out_hi + D, v);
    } else {
        cta_merge<Key, T>(A, K, B, K, out_hi, K, out_hi + K);
    }
}

// ------------------------------------------- quaternary merge path (q) --
// The per-level step is issue-bound (16 warps on 4 schedulers), so the merge
// minimises instructions per key: E = 8 outputs per thread amortise the split
// search, the search tests 3 points per round (latency of log4, instruction
// count of log2), and the thread's window is merged by an in-register bitonic
// network instead of a sequential merge.

// Largest i in [lo, hi] with P(i) = (i == lo || A[i-1] <= B[d-i]).
template <typename Key, int R>
__device__ __forceinline__ uint32_t split_q(const Key* __restrict__ A, const Key* __restrict__ B, uint32_t d,
                                            uint32_t na, uint32_t nb) {
    const uint32_t lo = d > nb ? d - nb : 0;
    const uint32_t hi = d < na ? d : na;
    uint32_t base = lo;
    // R = largest power of 4 <= range bound; reach 4R-1 >= range (see caller)
#pragma unroll
    for (uint32_t step = (uint32_t)R; step > 0; step >>= 2) {
        const uint32_t p1 = base + step, p2 = base + 2 * step, p3 = base + 3 * step;
        const uint32_t c = (uint32_t)(p1 <= hi && A[p1 - 1] <= B[d - p1]) +
                           (uint32_t)(p2 <= hi && A[p2 - 1] <= B[d - p2]) +
                           (uint32_t)(p3 <= hi && A[p3 - 1] <= B[d - p3]);
        base += c * step;
    }
    return base;
}

template <int N>
struct Pow4Floor {
    static constexpr int v = N >= 4 ? 4 * Pow4Floor<N / 4>::v : 1;
};
template <>
struct Pow4Floor<0> {
    static constexpr int v = 1;
};

// The E smallest of the windows A[i, i+E) and B[j, j+E) (sentinel-padded past
// na/nb), sorted, by a bitonic network in registers.
template <typename Key, int E>
__device__ __forceinline__ void window_first(const Key* __restrict__ A, uint32_t i, uint32_t na,
                                             const Key* __restrict__ B, uint32_t j, uint32_t nb,
                                             Key (&out)[E]) {
    Key x[2 * E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        x[e] = i + e < na ? A[i + e] : KeyLimits<Key>::kMax;
        x[2 * E - 1 - e] = j + e < nb ? B[j + e] : KeyLimits<Key>::kMax;
    }
    // bitonic split: the lower half becomes the E smallest
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const Key a = x[e], b = x[e + E];
        x[e] = a < b ? a : b;
    }
    // the lower half is bitonic: finish sorting it
#pragma unroll
    for (int st = E / 2; st >= 1; st >>= 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e & st) == 0) {
                const Key a = x[e], b = x[e + st];
                x[e] = a < b ? a : b;
                x[e + st] = a < b ? b : a;
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] = x[e];
}

// window_first with the windows fetched as 16-byte vectors: a warp's
// 16-byte loads at ~16-byte lane strides are bank-conflict-free, where scalar
// loads at 4-word strides conflict 4-way.  Reads up to 16 bytes past A+na /
// B+nb (callers pad shared memory).
template <typename Key, int E>
__device__ __forceinline__ void load_window_vec(const Key* __restrict__ A, uint32_t i, uint32_t na,
                                                Key (&x)[E]) {
    constexpr int KPC = 16 / (int)sizeof(Key);  // keys per chunk
    constexpr int C = E / KPC + 1;              // chunks covering E keys at any offset
    const uint4* v = reinterpret_cast<const uint4*>(A) + i / KPC;
    Key w[C * KPC];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const uint4 q = v[c];
        Key* d = w + c * KPC;
        if constexpr (KPC == 4) {
            d[0] = q.x; d[1] = q.y; d[2] = q.z; d[3] = q.w;
        } else {
            d[0] = ((unsigned long long)q.y << 32) | q.x;
            d[1] = ((unsigned long long)q.w << 32) | q.z;
        }
    }
    const uint32_t off = i % KPC;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        Key val;
        if constexpr (KPC == 4) {
            const Key lo2 = (off & 1u) ? w[e + 1] : w[e];
            const Key hi2 = (off & 1u) ? w[e + 3] : w[e + 2];
            val = (off & 2u) ? hi2 : lo2;
        } else {
            val = off ? w[e + 1] : w[e];
        }
        x[e] = i + e < na ? val : KeyLimits<Key>::kMax;
    }
}

template <typename Key, int E>
__device__ __forceinline__ void window_first_vec(const Key* __restrict__ A, uint32_t i, uint32_t na,
                                                 const Key* __restrict__ B, uint32_t j, uint32_t nb,
                                                 Key (&out)[E]) {
    Key a[E], b[E];
    load_window_vec<Key, E>(A, i, na, a);
    load_window_vec<Key, E>(B, j, nb, b);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const Key p = a[e], q = b[E - 1 - e];
        out[e] = p < q ? p : q;
    }
#pragma unroll
    for (int st = E / 2; st >= 1; st >>= 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e & st) == 0) {
                const Key p = out[e], q = out[e + st];
                out[e] = p < q ? p : q;
                out[e + st] = p < q ? q : p;
            }
        }
    }
}

template <int K, int T>
struct QShape {
    // outputs per thread: 8 when the CTA has enough threads for 2K/8, fewer
    // for tiny K, more when T is short
    static constexpr int kRaw = (2 * K + T - 1) / T;
    static constexpr int E = kRaw > 8 ? kRaw : (2 * K >= 8 * 32 ? 8 : (2 * K >= 4 * 8 ? 4 : 1));
    static constexpr int kActive = (2 * K) / E;
    static constexpr int kActiveHalf = K / E > 0 ? K / E : 1;
    static constexpr int R = Pow4Floor<K>::v;  // reach 4R-1 >= K
};

// merge_and_sort of two full K-batches (proj/src/batch.cpp:32-42): outputs
// [0,K) -> out_hi, [K,2K) -> out_lo, each half to shared memory or through L2.
template <typename Key, int K, int T, bool HiGlobal, bool LoGlobal>
__device__ __forceinline__ void cta_merge_q(const Key* __restrict__ A, const Key* __restrict__ B,
                                            Key* __restrict__ out_hi, Key* __restrict__ out_lo) {
    using Q = QShape<K, T>;
    constexpr int E = Q::E;
    if constexpr (E == 1 || (2 * K) % E != 0 || Q::kActive > T) {
        cta_merge_full<Key, K, T>(A, B, out_hi, out_lo);
    } else {
        const uint32_t d0 = threadIdx.x * E;
        if (d0 >= 2u * K) return;
        const uint32_t i = split_q<Key, Q::R>(A, B, d0, K, K);
        Key run[E];
        window_first<Key, E>(A, i, K, B, d0 - i, K, run);
        if (d0 < (uint32_t)K) {
            if constexpr (HiGlobal) store_run_cg<Key, E>(out_hi + d0, run);
            else store_run<Key, E>(out_hi + d0, run);
        } else {
            if constexpr (LoGlobal) store_run_cg<Key, E>(out_lo + (d0 - K), run);
            else store_run<Key, E>(out_lo + (d0 - K), run);
        }
    }
}

template <typename Key, int K, int T, bool HiGlobal, bool LoGlobal>
__device__ __forceinline__ void cta_merge_qv(const Key* __restrict__ A, const Key* __restrict__ B,
                                             Key* __restrict__ out_hi, Key* __restrict__ out_lo) {
    using Q = QShape<K, T>;
    constexpr int E = Q::E;
    if constexpr (E * sizeof(Key) < 16 || (2 * K) % E != 0 || Q::kActive > T) {
        cta_merge_full<Key, K, T>(A, B, out_hi, out_lo);
    } else {
        const uint32_t d0 = threadIdx.x * E;
        if (d0 >= 2u * K) return;
        const uint32_t i = split_q<Key, Q::R>(A, B, d0, K, K);
        Key run[E];
        window_first_vec<Key, E>(A, i, K, B, d0 - i, K, run);
        if (d0 < (uint32_t)K) {
            if constexpr (HiGlobal) store_run_cg<Key, E>(out_hi + d0, run);
            else store_run<Key, E>(out_hi + d0, run);
        } else {
            if constexpr (LoGlobal) store_run_cg<Key, E>(out_lo + (d0 - K), run);
            else store_run<Key, E>(out_lo + (d0 - K), run);
        }
    }
}

// First K outputs only.
template <typename Key, int K, int T, bool HiGlobal>
__device__ __forceinline__ void cta_merge_q_first(const Key* __restrict__ A, const Key* __restrict__ B,
                                                  Key* __restrict__ out_hi) {
    using Q = QShape<K, T>;
    constexpr int E = Q::E;
    if constexpr (E == 1 || K % E != 0 || Q::kActiveHalf > T) {
        cta_merge<Key, T>(A, K, B, K, out_hi, K, out_hi + K);
    } else {
        const uint32_t d0 = threadIdx.x * E;
        if (d0 >= (uint32_t)K) return;
        const uint32_t i = split_q<Key, Q::R>(A, B, d0, K, K);
        Key run[E];
        window_first<Key, E>(A, i, K, B, d0 - i, K, run);
        if constexpr (HiGlobal) store_run_cg<Key, E>(out_hi + d0, run);
        else store_run<Key, E>(out_hi + d0, run);
    }
}

// Block sort by merge passes: each thread sorts E keys in registers, then
// log2(K/E) rounds of pairwise run merges (quaternary splits, register
// windows) ping-pong between s and tmp.  Result in s.  Ends with a barrier.
template <typename Key, int K, int T>
__device__ __forceinline__ void cta_sort_merge(Key* __restrict__ s, Key* __restrict__ tmp) {
    constexpr int E = K >= 8 * 8 ? 8 : 1;
    constexpr int TS = K / E;
    if constexpr (E == 1 || TS > T) {
        cta_bitonic_sort<Key, K, T>(s);
    } else {
        const uint32_t t = threadIdx.x;
        if (t < (uint32_t)TS) {
            Key v[E];
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = s[t * E + e];
            // bitonic sort of E in registers
#pragma unroll
            for (int size = 2; size <= E; size <<= 1) {
#pragma unroll
                for (int st = size / 2; st >= 1; st >>= 1) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        if ((e & st) == 0) {
                            const bool up = (e & size) == 0;
                            const Key a = v[e], b = v[e + st];
                            const Key mn = a < b ? a : b, mx = a < b ? b : a;
                            v[e] = up ? mn : mx;
                            v[e + st] = up ? mx : mn;
                        }
                    }
                }
            }
            store_run<Key, E>(s + t * E, v);
        }
        __syncthreads();
        Key* src = s;
        Key* dst = tmp;
#pragma unroll 1
        for (uint32_t run = E; run < (uint32_t)K; run <<= 1) {
            if (t < (uint32_t)TS) {
                const uint32_t pair = (t * E) / (2 * run);
                const uint32_t d0 = t * E - pair * 2 * run;
                const Key* A = src + pair * 2 * run;
                const Key* B = A + run;
                // generic split (run varies): binary-then-quaternary over run
                const uint32_t lo = d0 > run ? d0 - run : 0;
                const uint32_t hi = d0 < run ? d0 : run;
                uint32_t base = lo;
                for (uint32_t step = Pow4Floor<K>::v; step > 0; step >>= 2) {
                    if (step > run) continue;
                    const uint32_t p1 = base + step, p2 = base + 2 * step, p3 = base + 3 * step;
                    base += step * ((uint32_t)(p1 <= hi && A[p1 - 1] <= B[d0 - p1]) +
                                    (uint32_t)(p2 <= hi && A[p2 - 1] <= B[d0 - p2]) +
                                    (uint32_t)(p3 <= hi && A[p3 - 1] <= B[d0 - p3]));
                }
                Key v[E];
                window_first<Key, E>(A, base, run, B, d0 - base, run, v);
                store_run<Key, E>(dst + pair * 2 * run + d0, v);
            }
            __syncthreads();
            Key* x = src;
            src = dst;
            dst = x;
        }
        if (src != s) {
            for (uint32_t i = t; i < (uint32_t)K; i += T) s[i] = src[i];
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ sort --
// Bitonic sort of K keys in shared memory with E keys per thread held in
// registers (blocked layout: thread t owns [t*E, t*E+E)).  Uses the first
// K/E threads; the rest only join the barriers.  Ends with a barrier; the
// sorted keys are back in s.
template <typename Key, int E>
__device__ __forceinline__ void cmpx(Key& a, Key& b, bool up) {
    const Key lo = a < b ? a : b;
    const Key hi = a < b ? b : a;
    a = up ? lo : hi;
    b = up ? hi : lo;
}

template <typename Key, int K, int T>
__device__ __forceinline__ void cta_sort_regs(Key* s) {
    constexpr int E = K >= 8 * 32 ? 8 : (K >= 64 ? 2 : 1);
    constexpr int TS = K / E;  // sorting threads
    static_assert(TS <= T || K < 64, "not enough threads for the register sort");
    if constexpr (K < 64 || TS > T) {
        cta_bitonic_sort<Key, K, T>(s);
    } else {
        const uint32_t t = threadIdx.x;
        const bool active = t < (uint32_t)TS;
        const uint32_t lane = t & 31;
        Key v[E];
        if (active) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = s[t * E + e];
        }
        constexpr uint32_t kWarpSpan = 32u * E;  // keys per warp
#pragma unroll 1
        for (uint32_t size = 2; size <= (uint32_t)K; size <<= 1) {
            uint32_t stride = size >> 1;
            // strides that cross warps: through shared memory
            if (stride >= kWarpSpan) {
                if (active) {
#pragma unroll
                    for (int e = 0; e < E; ++e) s[t * E + e] = v[e];
                }
                __syncthreads();
                for (; stride >= kWarpSpan; stride >>= 1) {
                    for (uint32_t p = t; p < (uint32_t)K / 2; p += T) {
                        const uint32_t i = 2 * p - (p & (stride - 1));
                        const uint32_t j = i + stride;
                        const bool up = (i & size) == 0;
                        const Key a = s[i], b = s[j];
                        if ((a > b) == up) {
                            s[i] = b;
                            s[j] = a;
                        }
                    }
                    __syncthreads();
                }
                if (active) {
#pragma unroll
                    for (int e = 0; e < E; ++e) v[e] = s[t * E + e];
                }
            }
            if (active) {
                // lane-crossing strides: partner lane = lane ^ (stride / E)
                for (; stride >= (uint32_t)E; stride >>= 1) {
                    const uint32_t lx = stride / E;
                    const bool lower = (lane & lx) == 0;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const uint32_t idx = t * E + e;
                        const bool up = (idx & size) == 0;
                        const Key o = __shfl_xor_sync(0xFFFFFFFFu, v[e], lx);
                        const Key mn = v[e] < o ? v[e] : o;
                        const Key mx = v[e] < o ? o : v[e];
                        v[e] = (lower == up) ? mn : mx;
                    }
                }
                // in-thread strides
#pragma unroll
                for (uint32_t st = E / 2; st > 0; st >>= 1) {
                    if (st > stride) continue;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        if ((e & st) == 0) {
                            const uint32_t idx = t * E + e;
                            const bool up = (idx & size) == 0;
                            cmpx<Key, E>(v[e], v[e + st], up);
                        }
                    }
                }
            }
        }
        if (active) {
#pragma unroll
            for (int e = 0; e < E; ++e) s[t * E + e] = v[e];
        }
        __syncthreads();
    }
}

}  // namespace bh

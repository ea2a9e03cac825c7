// bh_device.cuh -- CTA-level primitives of the batched generalized heap for
// sm_100a: multi-state node locks in HBM, coalesced node moves, the block
// bitonic sort and the merge-path MergeAndSort.
//
// One thread block owns one heap operation (section 4: "threads in
// one thread block work together for one INS and DEL operation"); lock words
// are driven by a single elected thread and the decision is broadcast through
// shared memory with a barrier, so warps never diverge on a lock.
#pragma once

#include <cstdint>

#include "bh_internal.h"

namespace bh {

template <typename Key>
struct KeyLimits;
template <>
struct KeyLimits<uint32_t> {
    static constexpr uint32_t kMax = 0xFFFFFFFFu;
};
template <>
struct KeyLimits<unsigned long long> {
    static constexpr unsigned long long kMax = ~0ull;
};

// ---------------------------------------------------------------- locks --
// GPU-scope acquire/release on the node state words (reference
// proj/src/heap.cpp:87-114 uses std::atomic acq_rel CAS + release store).
__device__ __forceinline__ uint32_t state_load(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Polling load without acquire semantics: ld.acquire.gpu invalidates the
// SM's L1 (CCTL.IVALL) on every poll, which stalls the shared-memory work
// of the other warps on the SM.  Spin with this, then acquire_fence() once
// the awaited word is seen (relaxed load + fence = acquire pattern).
__device__ __forceinline__ uint32_t state_poll(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void acquire_fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ bool state_cas(uint32_t* p, uint32_t expected, uint32_t desired) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;"
                 : "=r"(old)
                 : "l"(p), "r"(expected), "r"(desired)
                 : "memory");
    return old == expected;
}

// Relaxed claim CAS: the data ordering comes from the acquire poll that saw
// the holder's release, so the CAS only needs atomicity -- and, being
// relaxed, it does not hold back the node loads issued right after it (an
// acq_rel CAS would order them after its ~700-cycle round trip).
__device__ __forceinline__ bool state_cas_relaxed(uint32_t* p, uint32_t expected, uint32_t desired) {
    uint32_t old;
    asm volatile("atom.relaxed.gpu.global.cas.b32 %0, [%1], %2, %3;"
                 : "=r"(old)
                 : "l"(p), "r"(expected), "r"(desired)
                 : "memory");
    return old == expected;
}

__device__ __forceinline__ void state_store_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// A strong store with no ordering of its own: publishes data only when an
// explicit fence (__threadfence = fence.acq_rel.gpu) by the same thread has
// already ordered the CTA's writes before it.  (A red/st.release orders
// earlier writes before that one location only; it is not a fence for later
// relaxed stores.)
__device__ __forceinline__ void state_store_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Node state words carry a version above the 3-bit state: word = ver<<3 |
// state.  Claims CAS the exact observed word (state change, same version);
// every release bumps the version.  A claim that succeeds therefore proves
// the node did not change between the observation and the claim, which lets
// a CTA load a node's keys in the same round trip as the CAS that locks it.
__device__ __forceinline__ uint32_t sget(uint32_t w) { return w & 7u; }
__device__ __forceinline__ uint32_t swith(uint32_t w, uint32_t s) { return (w & ~7u) | s; }

// Release by the holder, who knows the state it holds (`from`): one
// red.release.gpu that bumps the version and moves the state to `to`.
__device__ __forceinline__ void state_release(uint32_t* p, uint32_t from, uint32_t to) {
    const uint32_t delta = 8u + to - from;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(delta) : "memory");
}

// The same transition without release semantics, for a hand-off that
// publishes no data (the gated BU park).
__device__ __forceinline__ void state_release_relaxed(uint32_t* p, uint32_t from, uint32_t to) {
    const uint32_t delta = 8u + to - from;
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(delta) : "memory");
}

// Warm L2 with n bytes at p (one prefetch per 128-byte line), issued by
// threads [first, first + lines).  A hint only: the later ld.cg of the lock
// holder reads whatever L2 holds then.
template <int T>
__device__ __forceinline__ void cta_prefetch_l2(const void* p, uint32_t bytes, uint32_t first) {
    const uint32_t lines = (bytes + 127) / 128;
    const uint32_t t = threadIdx.x - first;
    if (threadIdx.x >= first && t < lines) {
        const char* a = static_cast<const char*>(p) + t * 128;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
}

// Barrier of a thread group: id 0 is the whole CTA, ids 1..15 are named
// barriers over `nthr` threads (a multiple of 32).  Lets two halves of a CTA
// run independent protocol steps side by side.
__device__ __forceinline__ void grp_sync(uint32_t id, uint32_t nthr) {
    if (id == 0)
        __syncthreads();
    else
        asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthr) : "memory");
}

// ------------------------------------------------------------ mbarriers --
// Shared-memory mbarriers (sm_90+) for producer -> consumer hand-offs between
// the warp roles of a delete server (bh_heap.cuh, serve3): the producer's
// smem writes are released by its arrive, the consumer's wait acquires them.
// Phase n of a barrier completes after `count` arrivals; a consumer of the
// n-th completion waits for parity n & 1.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(unsigned long long* mb, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* mb) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mb)) : "memory");
}
__device__ __forceinline__ bool mb_test(unsigned long long* mb, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(mb)), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mb_wait(unsigned long long* mb, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(mb)), "r"(parity)
            : "memory");
    } while (!done);
}

// Group versions of the node moves (thread `tid` of `nthr`).
template <typename Key>
__device__ __forceinline__ void grp_load(Key* __restrict__ s, const Key* __restrict__ g, uint32_t n, uint32_t tid,
                                         uint32_t nthr) {
    const uint32_t bytes = n * (uint32_t)sizeof(Key);
    if (((bytes | (uint32_t)(uintptr_t)g) & 15u) == 0) {
        const uint4* gv = reinterpret_cast<const uint4*>(g);
        uint4* sv = reinterpret_cast<uint4*>(s);
        for (uint32_t i = tid; i < bytes / 16; i += nthr) sv[i] = __ldcg(gv + i);
    } else {
        for (uint32_t i = tid; i < n; i += nthr) s[i] = __ldcg(g + i);
    }
}

template <typename Key>
__device__ __forceinline__ void grp_store(Key* __restrict__ g, const Key* __restrict__ s, uint32_t n, uint32_t tid,
                                          uint32_t nthr) {
    const uint32_t bytes = n * (uint32_t)sizeof(Key);
    if (((bytes | (uint32_t)(uintptr_t)g) & 15u) == 0) {
        uint4* gv = reinterpret_cast<uint4*>(g);
        const uint4* sv = reinterpret_cast<const uint4*>(s);
        for (uint32_t i = tid; i < bytes / 16; i += nthr) __stcg(gv + i, sv[i]);
    } else {
        for (uint32_t i = tid; i < n; i += nthr) __stcg(g + i, s[i]);
    }
}

template <typename Key>
__device__ __forceinline__ void grp_fill_max(Key* g, uint32_t n, uint32_t tid, uint32_t nthr) {
    const uint32_t bytes = n * (uint32_t)sizeof(Key);
    if (((bytes | (uint32_t)(uintptr_t)g) & 15u) == 0) {
        uint4 fill;
        fill.x = fill.y = fill.z = fill.w = 0xFFFFFFFFu;
        uint4* gv = reinterpret_cast<uint4*>(g);
        for (uint32_t i = tid; i < bytes / 16; i += nthr) __stcg(gv + i, fill);
    } else {
        for (uint32_t i = tid; i < n; i += nthr) __stcg(g + i, ~Key(0));
    }
}

// Spin backoff (reference Backoff, proj/src/heap.cpp:18-31: 2^0..2^5 pause
// rounds, then yield).  On the GPU a waiting CTA sleeps in growing steps so the
// lock holder's SM and the contended L2 slice stay free.
// The first polls spin without sleeping: a lock hand-off on the critical
// path should cost one L2 round trip, not a sleep quantum.
// Device side of the deadlock watchdog (the reference's is a host thread,
// proj/src/workload.cpp:22-53): a wait that passes kStuckSpins pauses (about
// 4 s of 256 ns sleeps) raises a flag word (the heap header's error flags)
// once; the host watchdog of bh_run_ops reports it.
constexpr uint32_t kStuckSpins = 1u << 24;
constexpr unsigned long long kStuckFlag = 1ull << 4;  // = kErrStuck (bh_internal.h)
struct Backoff {
    uint32_t n = 0;
    unsigned long long* stuck = nullptr;
    __device__ __forceinline__ Backoff() {}
    __device__ __forceinline__ explicit Backoff(unsigned long long* flag_word) : stuck(flag_word) {}
    __device__ __forceinline__ void pause() {
        ++n;
        if (n > 32) __nanosleep(n > 64 ? 256 : 64);
        if (n == kStuckSpins && stuck) atomicOr(stuck, kStuckFlag);
    }
};
// For a waiter whose wake-up is on a critical path (a root queue-lock
// waiter, e.g. a delete that a delete server may hand a continuation): no
// sleep, each poll is one L2 round trip on the waiter's own 128-byte line
// (32 ns sleeps cost the 2^26 / K=1024 delete phase ~1.2 ms,
// profiles/r2/ab_final.txt).
struct QuickBackoff {
    uint32_t n = 0;
    unsigned long long* stuck = nullptr;
    __device__ __forceinline__ QuickBackoff() {}
    __device__ __forceinline__ explicit QuickBackoff(unsigned long long* flag_word) : stuck(flag_word) {}
    __device__ __forceinline__ void pause() {
        ++n;
        if (n == (kStuckSpins << 3) && stuck) atomicOr(stuck, kStuckFlag);
    }
};

// Asynchronous global -> shared copy of n keys (16-byte cp.async.cg, L2
// only); completes at cp_async_wait_all().  n * sizeof(Key) % 16 == 0.
template <typename Key, int T>
__device__ __forceinline__ void cta_load_async(Key* __restrict__ s, const Key* __restrict__ g, uint32_t n) {
    const uint32_t vecs = n * (uint32_t)sizeof(Key) / 16;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s);
    for (uint32_t i = threadIdx.x; i < vecs; i += T)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbase + 16 * i),
                     "l"(reinterpret_cast<const char*>(g) + 16ull * i)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ------------------------------------------------------------ L2 access --
// Heap data is shared across SMs whose L1s are not coherent: all node reads
// go through L2 (ld.global.cg) and all node writes are st.global.cg.
__device__ __forceinline__ unsigned long long ld_cg_u64(const unsigned long long* p) {
    return __ldcg(p);
}
__device__ __forceinline__ void st_cg_u64(unsigned long long* p, unsigned long long v) {
    __stcg(p, v);
}

template <typename Key>
__device__ __forceinline__ Key ld_key(const Key* p) {
    return __ldcg(p);
}
template <typename Key>
__device__ __forceinline__ void st_key(Key* p, Key v) {
    __stcg(p, v);
}

// CTA-cooperative copies of n keys.  16-byte vectors when both sides are
// aligned and the byte count is a multiple of 16 (always true for node copies
// with k*sizeof(Key) >= 16), scalar otherwise.  No barrier inside.
template <typename Key, int T>
__device__ __forceinline__ void cta_load(Key* __restrict__ s, const Key* __restrict__ g, uint32_t n) {
    const uint32_t bytes = n * (uint32_t)sizeof(Key);
    if (((bytes | (uint32_t)(uintptr_t)g) & 15u) == 0) {
        const uint4* gv = reinterpret_cast<const uint4*>(g);
        uint4* sv = reinterpret_cast<uint4*>(s);
        for (uint32_t i = threadIdx.x; i < bytes / 16; i += T) sv[i] = __ldcg(gv + i);
    } else {
        for (uint32_t i = threadIdx.x; i < n; i += T) s[i] = ld_key(g + i);
    }
}

template <typename Key, int T>
__device__ __forceinline__ void cta_store(Key* __restrict__ g, const Key* __restrict__ s, uint32_t n) {
    const uint32_t bytes = n * (uint32_t)sizeof(Key);
    if (((bytes | (uint32_t)(uintptr_t)g) & 15u) == 0) {
        uint4* gv = reinterpret_cast<uint4*>(g);
        const uint4* sv = reinterpret_cast<const uint4*>(s);
        for (uint32_t i = threadIdx.x; i < bytes / 16; i += T) __stcg(gv + i, sv[i]);
    } else {
        for (uint32_t i = threadIdx.x; i < n; i += T) st_key(g + i, s[i]);
    }
}

// Global -> global (partial buffer to a delete result).
template <typename Key, int T>
__device__ __forceinline__ void cta_copy_gg(Key* __restrict__ dst, const Key* __restrict__ src, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += T) st_key(dst + i, ld_key(src + i));
}

template <typename Key, int T>
__device__ __forceinline__ void cta_fill(Key* g, Key v, uint32_t n) {
    const uint32_t bytes = n * (uint32_t)sizeof(Key);
    if (((bytes | (uint32_t)(uintptr_t)g) & 15u) == 0) {
        uint4 fill;
        fill.x = fill.y = fill.z = fill.w = 0xFFFFFFFFu;  // v is always the all-ones sentinel
        uint4* gv = reinterpret_cast<uint4*>(g);
        for (uint32_t i = threadIdx.x; i < bytes / 16; i += T) __stcg(gv + i, fill);
    } else {
        for (uint32_t i = threadIdx.x; i < n; i += T) st_key(g + i, v);
    }
}

// ------------------------------------------------------------- sorting --
// Block bitonic sort of K keys in shared memory (section 4.1), every
// stage through shared memory with a CTA barrier.  Kept for node capacities
// below 32 (fewer keys than threads); cta_sort_batch below is the batch sort
// of every larger node.  Ends with a barrier.  Caller pads unused tail slots
// with the sentinel.
template <typename Key, int K, int T>
__device__ __forceinline__ void cta_bitonic_sort(Key* s) {
    if constexpr (K >= 2) {
        constexpr uint32_t kPairs = K / 2;
#pragma unroll 1
        for (uint32_t size = 2; size <= K; size <<= 1) {
#pragma unroll 1
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t p = threadIdx.x; p < kPairs; p += T) {
                    const uint32_t i = 2 * p - (p & (stride - 1));
                    const uint32_t j = i + stride;
                    const bool up = (i & size) == 0;
                    const Key a = s[i];
                    const Key b = s[j];
                    if ((a > b) == up) {
                        s[i] = b;
                        s[j] = a;
                    }
                }
                __syncthreads();
            }
        }
    } else {
        __syncthreads();
    }
}

// sort_batch (proj/src/batch.cpp:7-19) of one incoming batch: n <= K keys at
// g (global), sentinel-padded to K, sorted ascending into s0 (shared).  A
// register bitonic network: thread t holds keys [tE, tE + E), E = K / T,
// loaded as one E-key vector when aligned (8 or 16 bytes); compare-exchange
// stages of stride < E stay in the thread's registers, strides E..16E go
// through warp shuffles, and only strides >= 32E pass through shared memory,
// ping-ponging between s0 and s1 with one barrier per stage (10 of the 55
// stages at K = 1024, T = 512).  Returns, uniformly over the CTA, whether a
// key reached the sentinel (batch.cpp:13-15).  Ends with a barrier.
template <typename Key, int K, int T>
__device__ __forceinline__ bool cta_sort_batch(const Key* __restrict__ g, uint32_t n, Key* s0, Key* s1) {
    constexpr int E = K / T;
    static_assert(E >= 1 && E * T == K, "K must be a multiple of the CTA size");
    constexpr Key kMax = KeyLimits<Key>::kMax;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t base = threadIdx.x * E;
    Key v[E];
    constexpr uint32_t kVecBytes = E * sizeof(Key);
    const bool whole = base + E <= n;
    if constexpr (kVecBytes == 16 || kVecBytes == 8) {
        if (whole && ((uintptr_t)(g + base) % kVecBytes) == 0) {
            if constexpr (kVecBytes == 16) {
                const uint4 x = *reinterpret_cast<const uint4*>(g + base);
                const Key* px = reinterpret_cast<const Key*>(&x);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = px[e];
            } else {
                const uint2 x = *reinterpret_cast<const uint2*>(g + base);
                const Key* px = reinterpret_cast<const Key*>(&x);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = px[e];
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = base + e < n ? g[base + e] : kMax;
        }
    } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = base + e < n ? g[base + e] : kMax;
    }
    int bad = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) bad |= (base + e < n) && v[e] >= kMax;
    bad = __syncthreads_or(bad);
    if (bad) return true;
    uint32_t par = 0;
#pragma unroll
    for (uint32_t size = 2; size <= (uint32_t)K; size <<= 1) {
#pragma unroll
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32u * E) {  // partner in another warp
                Key* sb = par ? s1 : s0;
                par ^= 1u;
#pragma unroll
                for (int e = 0; e < E; ++e) sb[base + e] = v[e];
                __syncthreads();
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const uint32_t i = base + e;
                    const Key o = sb[i ^ stride];
                    const bool keep_min = ((i & stride) == 0) == ((i & size) == 0);
                    v[e] = keep_min ? (o < v[e] ? o : v[e]) : (o < v[e] ? v[e] : o);
                }
            } else if (stride >= (uint32_t)E) {  // partner in another lane of the warp
                const int d = (int)(stride / E);
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const uint32_t i = base + e;
                    const Key o = __shfl_xor_sync(0xFFFFFFFFu, v[e], d);
                    const bool keep_min = ((i & stride) == 0) == ((i & size) == 0);
                    v[e] = keep_min ? (o < v[e] ? o : v[e]) : (o < v[e] ? v[e] : o);
                }
            } else {  // partner in this thread's registers
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if ((e & (int)stride) == 0) {
                        const int f = e + (int)stride;
                        const bool up = ((base + e) & size) == 0;
                        const Key x = v[e], y = v[f];
                        const bool sw = up ? (y < x) : (x < y);
                        v[e] = sw ? y : x;
                        v[f] = sw ? x : y;
                    }
                }
            }
        }
    }
    (void)lane;
    __syncthreads();  // the last shared-memory stage's reads are done
#pragma unroll
    for (int e = 0; e < E; ++e) s0[base + e] = v[e];
    __syncthreads();
    return false;
}

// ------------------------------------------------------------- merging --
// Merge-path MergeAndSort (section 4.2, Odeh et al.): stable merge
// of sorted A[0,na) and B[0,nb) held in shared memory; output element d goes
// to out1[d] when d < split, else out2[d - split].  Ties take A first, as
// the reference's merge_sorted does (proj/src/batch.cpp:21-30).  Each thread
// binary-searches its diagonal, then merges its run in registers and writes
// it out.  No barrier inside.
template <typename Key, int T>
__device__ __forceinline__ void cta_merge(const Key* __restrict__ A, uint32_t na,
                                          const Key* __restrict__ B, uint32_t nb,
                                          Key* __restrict__ out1, uint32_t split,
                                          Key* __restrict__ out2) {
    const uint32_t total = na + nb;
    const uint32_t per = (total + T - 1) / T;
    const uint32_t d0 = threadIdx.x * per;
    if (d0 >= total) return;
    const uint32_t d1 = min(d0 + per, total);
    uint32_t lo = d0 > nb ? d0 - nb : 0;
    uint32_t hi = min(d0, na);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (A[mid] <= B[d0 - 1 - mid])
            lo = mid + 1;
        else
            hi = mid;
    }
    uint32_t i = lo, j = d0 - lo;
    for (uint32_t d = d0; d < d1; ++d) {
        const bool take_a = j >= nb || (i < na && A[i] <= B[j]);
        const Key v = take_a ? A[i++] : B[j++];
        if (d < split)
            out1[d] = v;
        else
            out2[d - split] = v;
    }
}

// Same contract, specialised for the hot case of two full k-batches with the
// split at k: each thread's run lies entirely in one output half, is built in
// registers and leaves as whole 16-byte vectors when aligned.
template <typename Key, int K, int T>
__device__ __forceinline__ void cta_merge_full(const Key* __restrict__ A, const Key* __restrict__ B,
                                               Key* __restrict__ out_hi, Key* __restrict__ out_lo) {
    constexpr uint32_t kTotal = 2 * K;
    constexpr uint32_t kPer = (kTotal + T - 1) / T;
    const uint32_t d0 = threadIdx.x * kPer;
    if (d0 >= kTotal) return;
    uint32_t lo = d0 > K ? d0 - K : 0;
    uint32_t hi = min(d0, (uint32_t)K);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (A[mid] <= B[d0 - 1 - mid])
            lo = mid + 1;
        else
            hi = mid;
    }
    uint32_t i = lo, j = d0 - lo;
    Key run[kPer];
#pragma unroll
    for (uint32_t e = 0; e < kPer; ++e) {
        const Key a = i < K ? A[i] : KeyLimits<Key>::kMax;
        const Key b = j < K ? B[j] : KeyLimits<Key>::kMax;
        const bool take_a = j >= K || (i < K && a <= b);
        run[e] = take_a ? a : b;
        i += take_a;
        j += !take_a;
    }
    Key* dst = d0 < K ? out_hi + d0 : out_lo + (d0 - K);
    constexpr uint32_t kRunBytes = kPer * sizeof(Key);
    if constexpr (kRunBytes % 16 == 0) {
        if (((uint32_t)(uintptr_t)dst & 15u) == 0) {
            uint4* dv = reinterpret_cast<uint4*>(dst);
            const uint4* rv = reinterpret_cast<const uint4*>(run);
#pragma unroll
            for (uint32_t v = 0; v < kRunBytes / 16; ++v) dv[v] = rv[v];
            return;
        }
    }
#pragma unroll
    for (uint32_t e = 0; e < kPer; ++e) dst[e] = run[e];
}

// needs_merge (proj/include/batchheap/batch.hpp:61-66) on two full batches in
// shared memory; every thread evaluates it identically.
template <typename Key, int K>
__device__ __forceinline__ bool needs_merge_full(const Key* a, const Key* b) {
    if (a[K - 1] <= b[0]) return false;
    if (b[K - 1] <= a[0]) return false;
    return true;
}

// ------------------------------------------------------------- bitrev ----
// proj/include/batchheap/bitrev.hpp:15-33 with the bit-reverse intrinsic.
__host__ __device__ __forceinline__ unsigned long long slot_for_rank(unsigned long long rank) {
#ifdef __CUDA_ARCH__
    const unsigned level = 63u - (unsigned)__clzll((long long)rank);
    const unsigned long long base = 1ull << level;
    const unsigned long long off = rank - base;
    return base + (level ? (__brevll(off) >> (64 - level)) : 0ull);
#else
    const unsigned level = 63u - (unsigned)__builtin_clzll(rank);
    const unsigned long long base = 1ull << level;
    unsigned long long off = rank - base, out = 0;
    for (unsigned i = 0; i < level; ++i) {
        out = (out << 1) | (off & 1);
        off >>= 1;
    }
    return base + out;
#endif
}

// Inverse of slot_for_rank (bit reversal is an involution within a level).
__host__ __device__ __forceinline__ unsigned long long rank_for_slot(unsigned long long slot) {
    return slot_for_rank(slot);
}

__device__ __forceinline__ unsigned level_of(unsigned long long slot) {
    return 63u - (unsigned)__clzll((long long)slot);
}

}  // namespace bh

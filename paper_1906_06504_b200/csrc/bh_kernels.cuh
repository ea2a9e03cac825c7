// bh_kernels.cuh -- kernel instantiation and launch dispatch for one key
// width.  Included by bh_kernels_u32.cu and bh_kernels_u64.cu with BH_KEY set.
#pragma once

#include <cuda_runtime.h>

#include "bh_heap.cuh"

namespace bh {

// Records a CUDA error for the C ABI's message; BH_OK on cudaSuccess.
int note_cuda(cudaError_t e);

// Standalone sort_batch over rows of stride K (proj/src/batch.cpp:7-19).
template <typename Key, int K, int T>
__global__ void __launch_bounds__(T) sort_rows_kernel(Key* keys, const uint32_t* lens,
                                                      unsigned long long rows) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Key* s = reinterpret_cast<Key*>(smem_raw);
    for (unsigned long long row = blockIdx.x; row < rows; row += gridDim.x) {
        Key* g = keys + row * K;
        const uint32_t n = lens ? lens[row] : (uint32_t)K;
        if constexpr (K >= T) {
            cta_sort_batch<Key, K, T>(g, n, s, s + K);  // (callers validated the keys)
        } else {
            for (uint32_t i = threadIdx.x; i < (uint32_t)K; i += T) s[i] = i < n ? g[i] : KeyLimits<Key>::kMax;
            __syncthreads();
            cta_bitonic_sort<Key, K, T>(s);
        }
        cta_store<Key, T>(g, s, K);
        __syncthreads();
    }
}

// Standalone merge_and_sort over row pairs (proj/src/batch.cpp:32-42).
template <typename Key, int K, int T>
__global__ void __launch_bounds__(T) merge_rows_kernel(const Key* a, const Key* b, Key* hi, Key* lo,
                                                       unsigned long long rows) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Key* sa = reinterpret_cast<Key*>(smem_raw);
    Key* sb = sa + K;
    for (unsigned long long row = blockIdx.x; row < rows; row += gridDim.x) {
        cta_load<Key, T>(sa, a + row * K, K);
        cta_load<Key, T>(sb, b + row * K, K);
        __syncthreads();
        cta_merge_full_bt<Key, K, T>(sa, sb, hi + row * K, lo + row * K);
        __syncthreads();
    }
}

// Quiescent invariant scan (check_invariants, proj/src/heap.cpp:726-770):
// one warp per slot.  result[0] = violation count, result[1] = first bad
// slot, result[2] = kind bitmask (1 state, 2 unoccupied-with-keys,
// 4 unsorted, 8 sentinel inside, 16 parent unoccupied, 32 property 1).
template <typename Key>
__global__ void check_kernel(HeapView hv, unsigned long long* result) {
    const Key kMax = KeyLimits<Key>::kMax;
    const uint32_t lane = threadIdx.x & 31;
    const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x / 32);
    const unsigned long long nodes = hv.hdr->node_count;
    const Key* keys = static_cast<const Key*>(hv.keys);
    const uint32_t k = hv.k;
    for (unsigned long long slot = 1 + (blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32);
         slot <= hv.slot_count; slot += warps) {
        uint32_t bad = 0;
        const Key* nd = keys + (slot - 1) * k;
        if (lane == 0 && (hv.states[slot * kStateStride] & 7u) != kAvail) bad |= 1;
        const bool occupied = rank_for_slot(slot) <= nodes;
        if (!occupied) {
            if (lane == 0 && nd[0] != kMax) bad |= 2;
        } else {
            for (uint32_t i = lane; i + 1 < k; i += 32)
                if (nd[i] > nd[i + 1]) bad |= 4;
            if (lane == 0 && nd[k - 1] == kMax) bad |= 8;
            if (lane == 0 && slot > 1) {
                if (rank_for_slot(slot / 2) > nodes)
                    bad |= 16;
                else if (nd[0] < keys[(slot / 2 - 1) * k + k - 1])
                    bad |= 32;
            }
        }
        bad = __reduce_or_sync(0xFFFFFFFFu, bad);
        if (lane == 0 && bad) {
            atomicAdd(&result[0], 1ull);
            atomicMin(&result[1], slot);
            atomicOr(&result[2], (unsigned long long)bad);
        }
    }
}

// collect_resident (proj/src/heap.cpp:716-724): ranks 1..nodes in order.
template <typename Key>
__global__ void gather_kernel(HeapView hv, unsigned long long nodes, Key* out) {
    const Key* keys = static_cast<const Key*>(hv.keys);
    const uint32_t k = hv.k;
    for (unsigned long long rank = 1 + blockIdx.x; rank <= nodes; rank += gridDim.x) {
        const Key* nd = keys + (slot_for_rank(rank) - 1) * k;
        for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) out[(rank - 1) * k + i] = nd[i];
    }
}

// SM count of the current device (grid sizes of the helper kernels).
inline int device_sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        return 1;
    return n;
}

template <typename Key, int K, bool Rec>
int launch_ops_kr(const HeapView& hv, const RunView& rv, uint32_t ctas, cudaStream_t stream) {
    using Cfg = KernelCfg<Key, K>;
    // (the dynamic shared memory attribute of both instantiations was set on
    // this device by bh_create through kernel_info_k)
    auto kern = heap_ops_kernel<Key, K, Cfg::kThreads, Rec>;
    kern<<<ctas, Cfg::kThreads, Cfg::kSmem, stream>>>(hv, rv);
    return note_cuda(cudaGetLastError());
}

// BH_FLAG_RECORD heaps run the kernel with the event log compiled in.
template <typename Key, int K>
int launch_ops_k(const HeapView& hv, const RunView& rv, uint32_t ctas, cudaStream_t stream) {
    if (hv.flags & BH_FLAG_RECORD) return launch_ops_kr<Key, K, true>(hv, rv, ctas, stream);
    return launch_ops_kr<Key, K, false>(hv, rv, ctas, stream);
}

template <typename Key, int K>
int kernel_info_k(KernelInfo* info) {
    using Cfg = KernelCfg<Key, K>;
    // Function attributes are per device: set them for both instantiations
    // (plain and recording) on the current device, which bh_create selected.
    auto kern = heap_ops_kernel<Key, K, Cfg::kThreads, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e != cudaSuccess) return note_cuda(e);
    e = cudaFuncSetAttribute(heap_ops_kernel<Key, K, Cfg::kThreads, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e != cudaSuccess) return note_cuda(e);
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, Cfg::kThreads, Cfg::kSmem) !=
        cudaSuccess)
        return BH_E_CUDA;
    info->threads = Cfg::kThreads;
    info->smem_bytes = Cfg::kSmem;
    info->max_ctas_per_sm = blocks;
    return BH_OK;
}

template <typename Key, int K>
int launch_sort_k(void* keys, const uint32_t* lens, uint64_t rows, cudaStream_t stream) {
    using Cfg = KernelCfg<Key, K>;
    const uint32_t smem = 2 * K * sizeof(Key);  // ping-pong pair of cta_sort_batch
    const unsigned long long cap = 16ull * device_sm_count();
    const unsigned grid = (unsigned)(rows < cap ? rows : cap);
    if (grid == 0) return BH_OK;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(sort_rows_kernel<Key, K, Cfg::kThreads>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return note_cuda(e);
    }
    sort_rows_kernel<Key, K, Cfg::kThreads>
        <<<grid, Cfg::kThreads, smem, stream>>>(static_cast<Key*>(keys), lens, rows);
    return note_cuda(cudaGetLastError());
}

template <typename Key, int K>
int launch_merge_k(const void* a, const void* b, void* hi, void* lo, uint64_t rows, cudaStream_t stream) {
    using Cfg = KernelCfg<Key, K>;
    const uint32_t smem = 2 * K * sizeof(Key);
    auto kern = merge_rows_kernel<Key, K, Cfg::kThreads>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return note_cuda(e);
    }
    const unsigned long long cap = 16ull * device_sm_count();
    const unsigned grid = (unsigned)(rows < cap ? rows : cap);
    if (grid == 0) return BH_OK;
    kern<<<grid, Cfg::kThreads, smem, stream>>>(static_cast<const Key*>(a), static_cast<const Key*>(b),
                                                static_cast<Key*>(hi), static_cast<Key*>(lo), rows);
    return note_cuda(cudaGetLastError());
}

#ifdef BH_DEV_KS  // development builds: a few node sizes only (fast compiles)
#define BH_FOR_EACH_K(X) X(2) X(32) X(256) X(1024)
#else
#define BH_FOR_EACH_K(X) \
    X(1) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048)
#endif

template <typename Key>
int dispatch_ops(const HeapView& hv, const RunView& rv, uint32_t ctas, cudaStream_t s) {
    switch (hv.k) {
#define X(KK) \
    case KK:  \
        return launch_ops_k<Key, KK>(hv, rv, ctas, s);
        BH_FOR_EACH_K(X)
#undef X
    }
    return BH_E_CONFIG;
}

template <typename Key>
int dispatch_info(uint32_t k, KernelInfo* info) {
    switch (k) {
#define X(KK) \
    case KK:  \
        return kernel_info_k<Key, KK>(info);
        BH_FOR_EACH_K(X)
#undef X
    }
    return BH_E_CONFIG;
}

template <typename Key>
int dispatch_sort(uint32_t k, void* keys, const uint32_t* lens, uint64_t rows, cudaStream_t s) {
    switch (k) {
#define X(KK) \
    case KK:  \
        return launch_sort_k<Key, KK>(keys, lens, rows, s);
        BH_FOR_EACH_K(X)
#undef X
    }
    return BH_E_CONFIG;
}

template <typename Key>
int dispatch_merge(uint32_t k, const void* a, const void* b, void* hi, void* lo, uint64_t rows,
                   cudaStream_t s) {
    switch (k) {
#define X(KK) \
    case KK:  \
        return launch_merge_k<Key, KK>(a, b, hi, lo, rows, s);
        BH_FOR_EACH_K(X)
#undef X
    }
    return BH_E_CONFIG;
}

template <typename Key>
int launch_check(const HeapView& hv, unsigned long long* result, cudaStream_t s) {
    check_kernel<Key><<<4 * device_sm_count(), 256, 0, s>>>(hv, result);
    return note_cuda(cudaGetLastError());
}

template <typename Key>
int launch_gather(const HeapView& hv, unsigned long long nodes, void* out, cudaStream_t s) {
    if (nodes == 0) return BH_OK;
    const unsigned long long cap = 8ull * device_sm_count();
    const unsigned grid = (unsigned)(nodes < cap ? nodes : cap);
    gather_kernel<Key><<<grid, 256, 0, s>>>(hv, nodes, static_cast<Key*>(out));
    return note_cuda(cudaGetLastError());
}

}  // namespace bh

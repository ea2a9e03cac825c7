// bh_apps.cu -- the heap's two application drivers:
//
//   * single-source shortest paths, proj/src/sssp.cpp:118-194: rounds of
//     "funnel the active set through the heap, take the nearest `threshold`
//     keys, relax them"; keys are dist<<32 | node in a 64-bit heap;
//   * 0/1 knapsack branch-and-bound, proj/src/knapsack.cpp:206-368: best-
//     first expansion of take/skip children with the fractional bound,
//     pruning against the shared best, and the drain-and-filter GC pass.
//
// Everything per-node runs on the device: the heap operations are bulk runs
// of the persistent heap kernel, relaxation / expansion / key encoding are
// kernels here, and the host loop only moves a few counters per round.  The
// reference runs the same loops on std::thread workers; the order in which
// nodes are explored differs, the results (exact distances, the optimum) do
// not.  The instance generators (grid_graph, generate_knapsack) restate the
// reference's with the same libstdc++ engines and distributions.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "bh_internal.h"

namespace {

constexpr unsigned long long kUnreachable = ~0ull;
constexpr unsigned long long kMaxEncodableDist = 0xFFFFFFFEull;  // sssp.cpp:14
constexpr unsigned long long kBenefitCeiling = 0xFFFFFFFEull;    // knapsack.cpp:175

int fail(int code, const std::string& msg) { return bh_internal_fail(code, msg.c_str()); }

#define APP_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) return fail(BH_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define APP_OK(call)                 \
    do {                             \
        int rc_ = (call);            \
        if (rc_ != BH_OK) return rc_; \
    } while (0)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    int alloc(size_t count) {
        if (count <= n) return BH_OK;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
        if (e != cudaSuccess) return fail(BH_E_CUDA, std::string("driver buffer: ") + cudaGetErrorString(e));
        n = std::max<size_t>(count, 1);
        return BH_OK;
    }
};

struct HeapGuard {
    bh_heap* h = nullptr;
    ~HeapGuard() {
        if (h) bh_destroy(h);
    }
};

struct StreamGuard {
    cudaStream_t s = nullptr;
    ~StreamGuard() {
        if (s) cudaStreamDestroy(s);
    }
};

inline unsigned long long sm_count_now() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        return 1;
    return (unsigned long long)n;
}

inline unsigned grid_for(unsigned long long n, unsigned threads = 256) {
    const unsigned long long g = (n + threads - 1) / threads;
    return (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>(g, 16ull * sm_count_now()));
}

// ------------------------------------------------------------------ SSSP --
struct Entry {  // sssp.cpp:22-25 ActiveEntry
    unsigned long long dist;
    uint32_t node;
    uint32_t pad;
};

__global__ void sssp_init(unsigned long long* dist, uint32_t n, uint32_t source, Entry* active) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        dist[v] = v == source ? 0ull : kUnreachable;
    if (blockIdx.x == 0 && threadIdx.x == 0) active[0] = Entry{0ull, source, 0u};
}

// encode (sssp.cpp:16-20): dist<<32 | node; an overflow sets err.
__global__ void sssp_encode(const Entry* a, unsigned long long n, unsigned long long* keys,
                            unsigned long long* err) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const Entry e = a[i];
        if (e.dist > kMaxEncodableDist) atomicOr(err, 1ull);
        keys[i] = (e.dist << 32) | e.node;
    }
}

// Popped batches (op i: lens[i] keys at out + i*k) -> entries, appended at
// *count (one reservation per batch).
__global__ void sssp_decode(const unsigned long long* out, const uint32_t* lens, unsigned long long n_ops,
                            uint32_t k, Entry* dst, unsigned long long* count) {
    for (unsigned long long op = blockIdx.x; op < n_ops; op += gridDim.x) {
        __shared__ unsigned long long base;
        const uint32_t len = lens[op];
        if (threadIdx.x == 0) base = len ? atomicAdd(count, (unsigned long long)len) : 0ull;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < len; j += blockDim.x) {
            const unsigned long long key = out[op * k + j];
            dst[base + j] = Entry{key >> 32, (uint32_t)key, 0u};
        }
        __syncthreads();
    }
}

// Relaxer::process (sssp.cpp:62-96): skip stale entries, relax every edge
// with an atomic min, append each improvement to `next`.
__global__ void sssp_relax(const Entry* set, unsigned long long n, const unsigned long long* off,
                           const uint32_t* nbr, const uint32_t* wgt, unsigned long long* dist, Entry* next,
                           unsigned long long* next_count, unsigned long long* visits) {
    unsigned long long my_visits = 0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const Entry e = set[i];
        if (e.dist > __ldcg(dist + e.node)) continue;  // stale
        ++my_visits;
        const unsigned long long b = off[e.node], f = off[e.node + 1];
        for (unsigned long long a = b; a < f; ++a) {
            const uint32_t v = nbr[a];
            const unsigned long long cand = e.dist + wgt[a];
            const unsigned long long seen = atomicMin(dist + v, cand);
            if (cand < seen) next[atomicAdd(next_count, 1ull)] = Entry{cand, v, 0u};
        }
    }
    if (my_visits) atomicAdd(visits, my_visits);
}

// ----------------------------------------------------------- knapsack --
struct BbNode {  // knapsack.cpp:127-132
    uint32_t level;
    uint32_t weight;
    uint32_t benefit;
    uint32_t bound;
};

// knapsack_bound (knapsack.cpp:106-123) over the density-sorted items.
__device__ unsigned long long bb_bound(const uint32_t* sw, const uint32_t* sb, uint32_t n, unsigned long long cap,
                                       uint32_t level, unsigned long long weight, unsigned long long benefit) {
    unsigned long long room = cap - weight;
    unsigned long long bound = benefit;
    for (uint32_t i = level; i < n; ++i) {
        const uint32_t w = sw[i];
        if (w <= room) {
            room -= w;
            bound += sb[i];
        } else {
            bound += room * sb[i] / w;  // fractional fill, floored
            break;
        }
    }
    return bound;
}

__device__ __forceinline__ unsigned long long bb_key(uint32_t benefit, uint32_t handle) {
    return ((kBenefitCeiling - benefit) << 32) | handle;  // encode_node, knapsack.cpp:177-180
}

struct BbDev {
    const uint32_t* sw;
    const uint32_t* sb;
    uint32_t n;
    unsigned long long cap;
    BbNode* arena;
    unsigned long long arena_cap;
    unsigned long long* arena_next;
    unsigned long long* best;
    unsigned long long* explored;
    unsigned long long* err;  // 1 = arena exhausted
    // Recycled slots: a stack of free handles.  The reference never frees
    // (its arena fills and the run terminates, knapsack.cpp:136-154); here
    // a popped node is dead once expanded (its children copy what they
    // need), so its slot is reused.  free_n is the stack height at kernel
    // start (fixed during a kernel), free_taken counts pops from the top.
    uint32_t* free_stack;
    unsigned long long* free_n;
    unsigned long long* free_taken;
    unsigned long long* free_pushed;
};

__device__ bool bb_alloc(const BbDev& d, const BbNode& node, uint32_t& handle) {
    const unsigned long long avail = *d.free_n;
    unsigned long long h;
    const unsigned long long idx = avail ? atomicAdd(d.free_taken, 1ull) : avail;
    if (idx < avail) {
        h = d.free_stack[avail - 1 - idx];
    } else {
        h = atomicAdd(d.arena_next, 1ull);
        if (h >= d.arena_cap) {
            atomicOr(d.err, 1ull);
            return false;
        }
    }
    d.arena[h] = node;
    handle = (uint32_t)h;
    return true;
}

// After a round: push the handles of every popped key (keep == nullptr) or
// of the drained keys GC dropped onto the free stack, above what the round
// left of it; bb_free_finish then settles the height.
__global__ void bb_free_popped(BbDev d, const unsigned long long* out, const uint32_t* lens, unsigned long long n_ops,
                               uint32_t k, bool gc_drop_only) {
    const unsigned long long total = n_ops * k;
    const unsigned long long avail = *d.free_n;
    const unsigned long long used = min(*d.free_taken, avail);
    const unsigned long long base = avail - used;
    const unsigned long long best_now = *d.best;
    for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < total;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        if ((uint32_t)(t % k) >= lens[t / k]) continue;
        const uint32_t h = (uint32_t)out[t];
        if (gc_drop_only && d.arena[h].bound > best_now) continue;  // kept by GC
        d.free_stack[base + atomicAdd(d.free_pushed, 1ull)] = h;
    }
}

__global__ void bb_free_finish(BbDev d) {
    const unsigned long long avail = *d.free_n;
    const unsigned long long used = min(*d.free_taken, avail);
    *d.free_n = avail - used + *d.free_pushed;
    *d.free_taken = 0;
    *d.free_pushed = 0;
}

// The worker loop body (knapsack.cpp:293-337) for every popped key: prune,
// take child (raises best), skip child, push survivors into `keys`.
__global__ void bb_expand(BbDev d, const unsigned long long* out, const uint32_t* lens, unsigned long long n_ops,
                          uint32_t k, unsigned long long* keys, unsigned long long* key_count) {
    const unsigned long long total = n_ops * k;
    for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < total;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long op = t / k;
        const uint32_t j = (uint32_t)(t % k);
        if (j >= lens[op]) continue;
        const uint32_t handle = (uint32_t)out[t];
        const BbNode node = d.arena[handle];
        const unsigned long long best_now = __ldcg(d.best);
        if (node.bound <= best_now || node.level >= d.n) continue;
        atomicAdd(d.explored, 1ull);
        const uint32_t wi = d.sw[node.level], bi = d.sb[node.level];
        const unsigned long long take_w = (unsigned long long)node.weight + wi;
        if (take_w <= d.cap) {
            BbNode take{node.level + 1, (uint32_t)take_w, node.benefit + bi, 0u};
            atomicMax(d.best, (unsigned long long)take.benefit);
            take.bound = (uint32_t)bb_bound(d.sw, d.sb, d.n, d.cap, take.level, take.weight, take.benefit);
            if (take.bound > __ldcg(d.best)) {
                uint32_t h;
                if (bb_alloc(d, take, h)) keys[atomicAdd(key_count, 1ull)] = bb_key(take.benefit, h);
            }
        }
        BbNode skip{node.level + 1, node.weight, node.benefit, 0u};
        skip.bound = (uint32_t)bb_bound(d.sw, d.sb, d.n, d.cap, skip.level, skip.weight, skip.benefit);
        if (skip.bound > __ldcg(d.best)) {
            uint32_t h;
            if (bb_alloc(d, skip, h)) keys[atomicAdd(key_count, 1ull)] = bb_key(skip.benefit, h);
        }
    }
}

// run_gc (knapsack.cpp:237-255): of the drained keys keep those whose node
// can still beat the best.
__global__ void bb_gc_filter(BbDev d, const unsigned long long* out, const uint32_t* lens, unsigned long long n_ops,
                             uint32_t k, unsigned long long* keys, unsigned long long* key_count) {
    const unsigned long long total = n_ops * k;
    const unsigned long long best_now = *d.best;
    for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < total;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        if ((uint32_t)(t % k) >= lens[t / k]) continue;
        const unsigned long long key = out[t];
        const BbNode node = d.arena[(uint32_t)key];
        if (node.bound > best_now) keys[atomicAdd(key_count, 1ull)] = key;
    }
}

// Bulk heap round: n_ops ops of `kind` planned on device, run, waited for.
struct HeapRunner {
    bh_heap* heap;
    cudaStream_t s;
    uint32_t k;
    uint32_t ctas;
    DevBuf<bh_op> ops;
    DevBuf<uint32_t> status, lens;
    int run(int kind, unsigned long long n_keys, const unsigned long long* pool, unsigned long long* out) {
        const unsigned long long n_ops = (n_keys + k - 1) / k;
        if (n_ops == 0) return BH_OK;
        APP_OK(ops.alloc(n_ops));
        APP_OK(status.alloc(n_ops));
        APP_OK(lens.alloc(n_ops));
        APP_OK(bh_plan_phase(heap, kind, n_keys, ops.p, 1, s));
        bh_run_cfg cfg{ctas, BH_RUN_EXPLICIT_STREAM, s};
        return bh_run_ops_device(heap, ops.p, n_ops, pool, out, status.p, lens.p, nullptr, &cfg);
    }
};

}  // namespace

// =================================================================== ABI ==
extern "C" {

uint64_t bh_grid_graph_edges(uint32_t rows, uint32_t cols) {
    if (rows == 0 || cols == 0) return 0;
    return 2ull * ((uint64_t)rows * (cols - 1) + (uint64_t)(rows - 1) * cols);
}

int bh_grid_graph(uint32_t rows, uint32_t cols, uint64_t seed, uint64_t* offsets, uint32_t* adj_node,
                  uint32_t* adj_weight) {
    if (!offsets || !adj_node || !adj_weight) return fail(BH_E_CONFIG, "null argument");
    const uint64_t n = (uint64_t)rows * cols;
    if (n == 0 || n > 0xFFFFFFFFull) return fail(BH_E_CONFIG, "grid size out of range");
    // Edge list in the reference's order (graph.cpp:174-193), then the CSR of
    // Graph::Graph (graph.cpp:12-30): counts per source, stable fill.
    struct E {
        uint32_t from, to, w;
    };
    std::vector<E> edges;
    edges.reserve(bh_grid_graph_edges(rows, cols));
    std::mt19937_64 rng(seed);
    auto weight = [&] { return std::uniform_int_distribution<uint32_t>(1, 1000)(rng); };
    auto id = [cols](uint32_t r, uint32_t c) { return r * cols + c; };
    for (uint32_t r = 0; r < rows; ++r) {
        for (uint32_t c = 0; c < cols; ++c) {
            if (c + 1 < cols) {
                const uint32_t w = weight();
                edges.push_back({id(r, c), id(r, c + 1), w});
                edges.push_back({id(r, c + 1), id(r, c), w});
            }
            if (r + 1 < rows) {
                const uint32_t w = weight();
                edges.push_back({id(r, c), id(r + 1, c), w});
                edges.push_back({id(r + 1, c), id(r, c), w});
            }
        }
    }
    std::fill(offsets, offsets + n + 1, 0ull);
    for (const E& e : edges) offsets[e.from + 1]++;
    for (uint64_t v = 0; v < n; ++v) offsets[v + 1] += offsets[v];
    std::vector<uint64_t> cursor(offsets, offsets + n);
    for (const E& e : edges) {
        const uint64_t at = cursor[e.from]++;
        adj_node[at] = e.to;
        adj_weight[at] = e.w;
    }
    return BH_OK;
}

int bh_sssp(uint32_t n_nodes, const uint64_t* offsets, const uint32_t* adj_node, const uint32_t* adj_weight,
            uint32_t source, const bh_sssp_cfg* cfg_in, int device, uint64_t* dist_out, bh_sssp_stats* stats) {
    if (!offsets || !adj_node || !adj_weight || !dist_out) return fail(BH_E_CONFIG, "null argument");
    if (source >= n_nodes) return fail(BH_E_CONFIG, "sssp: source out of range");
    // defaults: the reference's threshold; k = 1024 instead of the
    // reference's 32 (device ops are latency-bound per op, so wide nodes
    // win; distances do not depend on k)
    bh_sssp_cfg cfg = cfg_in ? *cfg_in : bh_sssp_cfg{10000, 1024, 0, 0};
    if (cfg.threshold == 0) cfg.threshold = 10000;
    if (cfg.heap_node_capacity == 0) cfg.heap_node_capacity = 1024;
    const uint32_t k = cfg.heap_node_capacity;
    const uint64_t m = offsets[n_nodes];
    const auto t0 = std::chrono::steady_clock::now();
    APP_CUDA(cudaSetDevice(device));
    StreamGuard sg;
    APP_CUDA(cudaStreamCreateWithFlags(&sg.s, cudaStreamNonBlocking));
    cudaStream_t s = sg.s;

    DevBuf<unsigned long long> d_off, d_dist, d_keys, d_out, d_ctr;
    DevBuf<uint32_t> d_nbr, d_wgt;
    DevBuf<Entry> d_active, d_proc;
    APP_OK(d_off.alloc(n_nodes + 1));
    APP_OK(d_nbr.alloc(m));
    APP_OK(d_wgt.alloc(m));
    APP_OK(d_dist.alloc(n_nodes));
    // the active set holds at most one entry per improvement of a round
    const uint64_t active_cap = m + n_nodes + 1;
    APP_OK(d_active.alloc(active_cap));
    APP_OK(d_keys.alloc(active_cap));
    const uint64_t want_cap = std::max<uint64_t>(cfg.threshold, k);
    const uint64_t proc_cap = std::max<uint64_t>(active_cap, (want_cap + k - 1) / k * k);
    APP_OK(d_proc.alloc(proc_cap));
    APP_OK(d_out.alloc((want_cap + k - 1) / k * k));
    APP_OK(d_ctr.alloc(4));  // 0 next count, 1 visits, 2 encode error, 3 popped count
    APP_CUDA(cudaMemcpyAsync(d_off.p, offsets, (n_nodes + 1) * 8, cudaMemcpyHostToDevice, s));
    APP_CUDA(cudaMemcpyAsync(d_nbr.p, adj_node, m * 4, cudaMemcpyHostToDevice, s));
    APP_CUDA(cudaMemcpyAsync(d_wgt.p, adj_weight, m * 4, cudaMemcpyHostToDevice, s));
    APP_CUDA(cudaMemsetAsync(d_ctr.p, 0, 4 * 8, s));
    sssp_init<<<grid_for(n_nodes), 256, 0, s>>>(d_dist.p, n_nodes, source, d_active.p);
    APP_CUDA(cudaGetLastError());

    // sssp.cpp:122-125: BU heap, k, max_nodes sized for the edge count
    const uint64_t max_nodes = std::max<uint64_t>(1024, (m + n_nodes) * 4 / k + 64);
    if (max_nodes > (1ull << 30)) return fail(BH_E_CONFIG, "sssp: graph too large for the heap");
    HeapGuard hg;
    APP_OK(bh_create(&hg.h, BH_BU, k, (uint32_t)max_nodes, 64, BH_FLAG_ELIDE_MERGES, device));
    HeapRunner hr{hg.h, s, k, cfg.ctas};

    uint64_t active_n = 1, pending = 0, visits_rounds = 0, rounds = 0, through = 0;
    unsigned long long h_ctr[4];
    while (active_n > 0 || pending > 0) {
        uint64_t proc_n;
        if (pending == 0 && active_n <= cfg.threshold) {
            std::swap(d_active.p, d_proc.p);
            std::swap(d_active.n, d_proc.n);
            proc_n = active_n;
        } else {
            // funnel the active set through the heap (sssp.cpp:135-150)
            sssp_encode<<<grid_for(active_n), 256, 0, s>>>(d_active.p, active_n, d_keys.p, d_ctr.p + 2);
            APP_CUDA(cudaGetLastError());
            APP_OK(hr.run(0, active_n, d_keys.p, nullptr));
            pending += active_n;
            through += active_n;
            // take the nearest max(threshold, k) keys (sssp.cpp:152-177)
            const uint64_t want = std::min<uint64_t>(pending, want_cap);
            const uint64_t n_del = (want + k - 1) / k;
            APP_CUDA(cudaMemsetAsync(d_ctr.p + 3, 0, 8, s));
            APP_OK(hr.run(1, n_del * k, nullptr, d_out.p));
            sssp_decode<<<(unsigned)std::min<uint64_t>(n_del, 8ull * sm_count_now()), 128, 0, s>>>(d_out.p, hr.lens.p, n_del, k,
                                                                                  d_proc.p, d_ctr.p + 3);
            APP_CUDA(cudaGetLastError());
            APP_CUDA(cudaMemcpyAsync(h_ctr + 3, d_ctr.p + 3, 8, cudaMemcpyDeviceToHost, s));
            APP_CUDA(cudaStreamSynchronize(s));
            proc_n = h_ctr[3];
            pending -= proc_n;
        }
        // relax; the improvements become the next active set
        APP_CUDA(cudaMemsetAsync(d_ctr.p, 0, 8, s));
        if (proc_n)
            sssp_relax<<<grid_for(proc_n), 256, 0, s>>>(d_proc.p, proc_n, d_off.p, d_nbr.p, d_wgt.p, d_dist.p,
                                                         d_active.p, d_ctr.p, d_ctr.p + 1);
        APP_CUDA(cudaGetLastError());
        APP_CUDA(cudaMemcpyAsync(h_ctr, d_ctr.p, 3 * 8, cudaMemcpyDeviceToHost, s));
        APP_CUDA(cudaStreamSynchronize(s));
        if (h_ctr[2]) return fail(BH_E_INVALID_KEY, "sssp: distance exceeds encodable range");
        active_n = h_ctr[0];
        visits_rounds = h_ctr[1];
        ++rounds;
    }
    APP_CUDA(cudaMemcpyAsync(dist_out, d_dist.p, (uint64_t)n_nodes * 8, cudaMemcpyDeviceToHost, s));
    APP_CUDA(cudaStreamSynchronize(s));
    if (stats) {
        stats->visits = visits_rounds;
        stats->rounds = rounds;
        stats->keys_through_heap = through;
        stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    return BH_OK;
}

uint64_t bh_generate_knapsack(int type, uint32_t n, uint32_t range, uint64_t seed, uint32_t* weight,
                              uint32_t* benefit) {
    // generate_knapsack (knapsack.cpp:22-66)
    if (n < 1 || range < 10 || !weight || !benefit || type < 0 || type > 3) {
        fail(BH_E_CONFIG, "knapsack generator needs n >= 1 and range >= 10");
        return 0;
    }
    std::mt19937_64 rng(seed);
    const uint32_t shift = range / 10;
    const uint32_t band = range / 500;
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t w = std::uniform_int_distribution<uint32_t>(1, range)(rng);
        uint32_t b = 0;
        switch (type) {
            case BH_KS_STRONGLY_CORRELATED:
                b = w + shift;
                break;
            case BH_KS_ALMOST_STRONGLY_CORRELATED: {
                const uint32_t lo = (w + shift > band) ? w + shift - band : 1;
                b = std::uniform_int_distribution<uint32_t>(lo, w + shift + band)(rng);
                break;
            }
            case BH_KS_EVEN_ODD:
                w = 2 * std::uniform_int_distribution<uint32_t>(1, std::max(1u, range / 2))(rng);
                b = w + shift;
                break;
            default:  // subset sum
                b = w;
                break;
        }
        weight[i] = w;
        benefit[i] = b;
    }
    uint64_t capacity = (uint64_t)n * range / 4;
    if (type == BH_KS_EVEN_ODD) capacity |= 1;  // odd W
    return capacity;
}

int bh_knapsack_bb(uint32_t n, const uint32_t* weight, const uint32_t* benefit, uint64_t capacity,
                   const bh_bb_cfg* cfg_in, int device, bh_bb_outcome* outcome) {
    if (!weight || !benefit || !outcome) return fail(BH_E_CONFIG, "null argument");
    if (n < 1) return fail(BH_E_CONFIG, "empty knapsack instance");
    if (capacity > 0xFFFFFFFFull) return fail(BH_E_CONFIG, "knapsack capacity exceeds 32-bit node fields");
    // defaults tuned for the device (tools/apps_sweep.py): k = 1024, four
    // batches per round, GC at 2^20 keys (reference: k = 32, 2 workers, GC
    // at 2^16); the optimum does not depend on them
    bh_bb_cfg cfg = cfg_in ? *cfg_in : bh_bb_cfg{1u << 20, 1024, 0, 4, 0, 0, 0};
    if (cfg.max_explored == 0) cfg.max_explored = 1ull << 29;
    if (cfg.heap_node_capacity == 0) cfg.heap_node_capacity = 1024;
    if (cfg.pop_ops == 0) cfg.pop_ops = 4;
    if (cfg.arena_nodes == 0) cfg.arena_nodes = 1ull << 28;  // 4 GiB of 16-byte nodes
    const uint32_t k = cfg.heap_node_capacity;
    const auto t0 = std::chrono::steady_clock::now();

    // density_sorted (knapsack.cpp:81-104): decreasing b/w, index tie-break
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        const uint64_t lhs = (uint64_t)benefit[a] * weight[b];
        const uint64_t rhs = (uint64_t)benefit[b] * weight[a];
        if (lhs != rhs) return lhs > rhs;
        return a < b;
    });
    std::vector<uint32_t> sw(n), sb(n);
    for (uint32_t i = 0; i < n; ++i) {
        sw[i] = weight[order[i]];
        sb[i] = benefit[order[i]];
    }
    // root bound on the host (the same fractional relaxation)
    uint64_t root_bound = 0;
    {
        uint64_t room = capacity;
        for (uint32_t i = 0; i < n; ++i) {
            if (sw[i] <= room) {
                room -= sw[i];
                root_bound += sb[i];
            } else {
                root_bound += room * sb[i] / sw[i];
                break;
            }
        }
    }
    if (root_bound > kBenefitCeiling) return fail(BH_E_CONFIG, "knapsack benefits exceed the key encoding");

    APP_CUDA(cudaSetDevice(device));
    StreamGuard sg;
    APP_CUDA(cudaStreamCreateWithFlags(&sg.s, cudaStreamNonBlocking));
    cudaStream_t s = sg.s;
    DevBuf<uint32_t> d_sw, d_sb;
    DevBuf<BbNode> d_arena;
    DevBuf<unsigned long long> d_ctr, d_keys, d_out;
    APP_OK(d_sw.alloc(n));
    APP_OK(d_sb.alloc(n));
    APP_OK(d_arena.alloc(cfg.arena_nodes));
    DevBuf<uint32_t> d_free;
    APP_OK(d_free.alloc(cfg.arena_nodes));
    APP_OK(d_ctr.alloc(8));  // 0 arena_next, 1 best, 2 explored, 3 err, 4 key count, 5-7 free stack
    APP_CUDA(cudaMemcpyAsync(d_sw.p, sw.data(), n * 4, cudaMemcpyHostToDevice, s));
    APP_CUDA(cudaMemcpyAsync(d_sb.p, sb.data(), n * 4, cudaMemcpyHostToDevice, s));
    unsigned long long init[8] = {1, 0, 0, 0, 1, 0, 0, 0};  // arena slot 0 = the root
    APP_CUDA(cudaMemcpyAsync(d_ctr.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
    const BbNode root{0, 0, 0, (uint32_t)root_bound};
    APP_CUDA(cudaMemcpyAsync(d_arena.p, &root, sizeof(root), cudaMemcpyHostToDevice, s));

    // knapsack.cpp:213: BU heap of k-key nodes; sized for the GC threshold
    // plus one round of children
    const uint64_t pop_keys = (uint64_t)cfg.pop_ops * k;
    const uint64_t key_cap = std::max<uint64_t>(2 * pop_keys, cfg.gc_threshold ? cfg.gc_threshold : (1ull << 20)) +
                             2 * pop_keys + k;
    uint64_t max_nodes = std::max<uint64_t>(1u << 18, 4 * (key_cap / k + 64));
    if (max_nodes > (1ull << 30)) max_nodes = 1ull << 30;
    HeapGuard hg;
    APP_OK(bh_create(&hg.h, BH_BU, k, (uint32_t)max_nodes, 64, BH_FLAG_ELIDE_MERGES, device));
    HeapRunner hr{hg.h, s, k, cfg.ctas};
    APP_OK(d_keys.alloc(std::max<uint64_t>(2 * pop_keys, 1024)));
    APP_OK(d_out.alloc(pop_keys));
    BbDev dv{d_sw.p,      d_sb.p,      n,           capacity,   d_arena.p,  cfg.arena_nodes, d_ctr.p, d_ctr.p + 1,
             d_ctr.p + 2, d_ctr.p + 3, d_free.p,   d_ctr.p + 5, d_ctr.p + 6, d_ctr.p + 7};

    // the root key
    {
        const unsigned long long key = ((kBenefitCeiling - 0ull) << 32) | 0ull;
        APP_CUDA(cudaMemcpyAsync(d_keys.p, &key, 8, cudaMemcpyHostToDevice, s));
        APP_OK(hr.run(0, 1, d_keys.p, nullptr));
    }
    uint64_t rounds = 0, gc_passes = 0, in_heap = 1;
    unsigned long long h_ctr[8];
    while (in_heap > 0) {
        // pop a round of best-first batches (the workers' try_delete_min)
        const uint64_t n_del = std::min<uint64_t>(cfg.pop_ops, (in_heap + k - 1) / k + 1);
        APP_CUDA(cudaMemsetAsync(d_ctr.p + 4, 0, 8, s));
        APP_OK(hr.run(1, n_del * k, nullptr, d_out.p));
        bb_expand<<<grid_for(n_del * k), 256, 0, s>>>(dv, d_out.p, hr.lens.p, n_del, k, d_keys.p, d_ctr.p + 4);
        APP_CUDA(cudaGetLastError());
        bb_free_popped<<<grid_for(n_del * k), 256, 0, s>>>(dv, d_out.p, hr.lens.p, n_del, k, false);
        bb_free_finish<<<1, 1, 0, s>>>(dv);
        APP_CUDA(cudaGetLastError());
        APP_CUDA(cudaMemcpyAsync(h_ctr, d_ctr.p, 8 * 8, cudaMemcpyDeviceToHost, s));
        APP_CUDA(cudaStreamSynchronize(s));
        if (h_ctr[3]) return fail(BH_E_CAPACITY, "branch-and-bound arena exhausted");
        if (h_ctr[2] > cfg.max_explored) return fail(BH_E_CAPACITY, "branch-and-bound node budget exhausted");
        const uint64_t pushed = h_ctr[4];
        APP_OK(hr.run(0, pushed, d_keys.p, nullptr));
        bh_peek pk;
        APP_CUDA(cudaStreamSynchronize(s));
        APP_OK(bh_peek_stats(hg.h, &pk));
        in_heap = pk.key_count;
        ++rounds;
        // GC (knapsack.cpp:237-255, 339-345): drain, filter, reinsert
        if (cfg.gc_threshold > 0 && in_heap > cfg.gc_threshold) {
            const uint64_t drain_ops = (in_heap + k - 1) / k + 1;
            APP_OK(d_out.alloc(drain_ops * k));
            APP_OK(d_keys.alloc(std::max<uint64_t>(drain_ops * k, 2 * pop_keys)));
            APP_CUDA(cudaMemsetAsync(d_ctr.p + 4, 0, 8, s));
            APP_OK(hr.run(1, drain_ops * k, nullptr, d_out.p));
            bb_gc_filter<<<grid_for(drain_ops * k), 256, 0, s>>>(dv, d_out.p, hr.lens.p, drain_ops, k, d_keys.p,
                                                                  d_ctr.p + 4);
            bb_free_popped<<<grid_for(drain_ops * k), 256, 0, s>>>(dv, d_out.p, hr.lens.p, drain_ops, k, true);
            bb_free_finish<<<1, 1, 0, s>>>(dv);
            APP_CUDA(cudaGetLastError());
            APP_CUDA(cudaMemcpyAsync(h_ctr + 4, d_ctr.p + 4, 8, cudaMemcpyDeviceToHost, s));
            APP_CUDA(cudaStreamSynchronize(s));
            APP_OK(hr.run(0, h_ctr[4], d_keys.p, nullptr));
            APP_CUDA(cudaStreamSynchronize(s));
            APP_OK(bh_peek_stats(hg.h, &pk));
            in_heap = pk.key_count;
            ++gc_passes;
        }
    }
    APP_CUDA(cudaMemcpyAsync(h_ctr, d_ctr.p, 8 * 8, cudaMemcpyDeviceToHost, s));
    APP_CUDA(cudaStreamSynchronize(s));
    outcome->best = h_ctr[1];
    outcome->explored = h_ctr[2];
    outcome->gc_passes = gc_passes;
    outcome->rounds = rounds;
    outcome->arena_nodes = h_ctr[0];  // slots ever used (high-water mark)
    outcome->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return BH_OK;
}

}  // extern "C"

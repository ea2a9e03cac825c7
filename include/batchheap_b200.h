/*
 * batchheap_b200.h -- C ABI of the B200-native batched generalized heap.
 *
 * This is the drop-in boundary for the reference's hot path, the C++ class
 * batchheap::GeneralizedHeap (reference proj/include/batchheap/heap.hpp:72-181,
 * proj/src/heap.cpp).  Plain pointers and sizes only; no exceptions or torch
 * types cross it.  Every entry point names the reference interface it
 * replaces.  The C++ facade in include/batchheap_b200.hpp rebuilds the
 * reference's class shape (methods, exception types) on top of these calls.
 *
 * Keys are unsigned integers of the handle's width (32 or 64 bits).  The
 * largest value of that width is the reserved empty-slot sentinel
 * (reference kMaxKey, proj/include/batchheap/batch.hpp:17-21); user keys must
 * be strictly smaller.
 */
#ifndef BATCHHEAP_B200_H
#define BATCHHEAP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BH_API __attribute__((visibility("default")))

/* Status codes.  The reference throws; the ABI returns.
 *   BH_E_CONFIG       <- ConfigError        (proj/include/batchheap/batch.hpp:23-25)
 *   BH_E_CAPACITY     <- CapacityError      (proj/include/batchheap/batch.hpp:26-28)
 *   BH_E_EMPTY        <- EmptyHeapError / try_delete_min()==nullopt (:29-31)
 *   BH_E_INVALID_KEY  <- std::invalid_argument "key reaches sentinel" (proj/src/batch.cpp:13-15)
 *   BH_E_CUDA         -- device/runtime failure (no reference analogue)
 *   BH_E_INTERNAL     -- protocol invariant broken (reference std::logic_error,
 *                        proj/src/heap.cpp:462-463); the synchronous entry
 *                        points (bh_insert, bh_delete_min, bh_run_ops) check
 *                        the device fault flags after every call             */
enum {
    BH_OK = 0,
    BH_E_CONFIG = 1,
    BH_E_CAPACITY = 2,
    BH_E_EMPTY = 3,
    BH_E_INVALID_KEY = 4,
    BH_E_CUDA = 5,
    BH_E_INTERNAL = 6
};

/* Protocol variant (reference enum class Variant, proj/include/batchheap/history.hpp:23). */
enum { BH_TD = 0, BH_BU = 1 };

/* bh_create flags. */
#define BH_FLAG_ELIDE_MERGES 0x1u /* HeapOptions::elide_merges (heap.hpp:43-47); default on */
#define BH_FLAG_RECORD 0x2u       /* device event log for linearizability checks (Recorder*) */
#define BH_FLAG_PROFILE 0x4u      /* per-phase SM-cycle counters (bh_profile) */

typedef struct bh_heap bh_heap;

/* HeapPeek (proj/include/batchheap/heap.hpp:60-65). */
typedef struct {
    uint64_t node_count;
    uint64_t key_count;
    uint64_t partial_len;
    uint64_t level_count;
} bh_peek;

/* HeapCounters (proj/include/batchheap/heap.hpp:49-58), same field order. */
typedef struct {
    uint64_t inserts;
    uint64_t deletes;
    uint64_t merges;
    uint64_t elided_merges;
    uint64_t early_stops;
    uint64_t propagation_node_visits;
    uint64_t coop_handoffs;
    uint64_t max_partial_len;
} bh_counters;

/* One operation of a bulk submission. */
enum { BH_OP_INSERT = 0, BH_OP_DELETE = 1 };
typedef struct {
    uint32_t kind;   /* BH_OP_INSERT / BH_OP_DELETE */
    uint32_t len;    /* insert: number of keys, 1..k; delete: ignored */
    uint64_t offset; /* insert: first key in key_pool; delete: first slot (k wide) in out_pool */
} bh_op;

/* Launch configuration of a bulk run. */
#define BH_RUN_EXPLICIT_STREAM 0x1u /* use cfg->stream even when NULL (legacy default stream) */
typedef struct {
    uint32_t ctas;   /* persistent CTAs; 0 = all co-resident CTAs the device holds */
    uint32_t flags;  /* BH_RUN_* */
    void* stream;    /* cudaStream_t; NULL = the handle's own stream unless BH_RUN_EXPLICIT_STREAM */
} bh_run_cfg;

/* ---------------------------------------------------------------------------
 * Lifecycle.  Replaces GeneralizedHeap(Variant, uint32 k, uint32 max_nodes,
 * HeapOptions, Recorder*) (proj/include/batchheap/heap.hpp:74-75,
 * proj/src/heap.cpp:42-62).  k must be a power of two in [1, 2048] (the
 * reference stops at 1024, proj/include/batchheap/batch.hpp:34-36; 2048 is a
 * deliberate extension for the K-sweep); max_nodes in [1, 2^30]; key_bits 32
 * or 64.  The handle owns all device memory on `device`.
 * ------------------------------------------------------------------------- */
BH_API int bh_create(bh_heap** out, int variant, uint32_t k, uint32_t max_nodes,
                     uint32_t key_bits, uint32_t flags, int device);
BH_API void bh_destroy(bh_heap* heap);

/* GeneralizedHeap::insert(std::span<const Key>) (heap.hpp:81-83, heap.cpp:123-188).
 * Copies 1..k caller keys (host memory).  BH_E_CAPACITY when n is 0 or > k,
 * or (before any mutation) when a full batch is needed and the heap is full;
 * BH_E_INVALID_KEY when a key reaches the sentinel.  Safe to call from many
 * host threads at once: each call runs as its own device operation and the
 * ops synchronize through the per-node device locks. */
BH_API int bh_insert(bh_heap* heap, const void* keys, uint32_t n);

/* GeneralizedHeap::delete_min() / try_delete_min() (heap.hpp:86-88,
 * heap.cpp:411-465).  Writes the k smallest keys at the linearization point
 * (fewer when fewer remain) into `out` (host, capacity >= k); BH_E_EMPTY
 * replaces both the EmptyHeapError throw and the nullopt return. */
BH_API int bh_delete_min(bh_heap* heap, void* out, uint32_t* n_out);

/* Bulk path (new; the reference issues ops from host threads,
 * proj/src/bench.cpp:78-124).  Executes n_ops operations concurrently in one
 * persistent-kernel launch, each CTA owning one op at a time, linearizable
 * exactly as concurrent host callers would be.  Host buffers; the call copies
 * in, runs and copies out before returning.  out_status/out_lens/out_seq may
 * be NULL.  out_seq[i] is the op's root-lock sequence number (the order in
 * which ops held the root: the TD linearization order, and the delete order
 * for BU). */
BH_API int bh_run_ops(bh_heap* heap, const bh_op* ops, uint64_t n_ops, const void* key_pool,
                      uint64_t key_pool_len, void* out_pool, uint64_t out_pool_len,
                      uint32_t* out_status, uint32_t* out_lens, uint64_t* out_seq,
                      const bh_run_cfg* cfg);

/* Same with DEVICE pointers (all arrays already resident), asynchronous on
 * cfg->stream.  The bench's kernel-only path. */
BH_API int bh_run_ops_device(bh_heap* heap, const bh_op* ops, uint64_t n_ops,
                             const void* key_pool, void* out_pool, uint32_t* out_status,
                             uint32_t* out_lens, uint64_t* out_seq, const bh_run_cfg* cfg);

/* Fills `ops` (host or device per `on_device`) with the phase-separated plan
 * used by the benchmark: n_keys keys in batches of k (last one partial) as
 * inserts, or ceil(n_keys/k) deletes writing k-wide slots. */
BH_API int bh_plan_phase(bh_heap* heap, int kind, uint64_t n_keys, bh_op* ops, int on_device,
                         void* stream);

/* ---------------------------------------------------------------------------
 * Introspection.  peek_stats is a racy monitoring snapshot; the rest require
 * quiescence (no bulk run or call in flight), as in the reference
 * (heap.hpp:25-26,90-104).
 * ------------------------------------------------------------------------- */
BH_API int bh_peek_stats(bh_heap* heap, bh_peek* out);                 /* peek_stats()  heap.cpp:671-678 */
BH_API int bh_get_counters(bh_heap* heap, bh_counters* out);           /* counters()    heap.cpp:680-697 */
BH_API int bh_reset_counters(bh_heap* heap);                           /* reset_counters() heap.cpp:699-708 */
BH_API int bh_select_insert_target(bh_heap* heap, uint64_t* slot);     /* select_insert_target() heap.cpp:710-714 */
BH_API int bh_collect_resident(bh_heap* heap, void* out, uint64_t cap, /* collect_resident() heap.cpp:716-724 */
                               uint64_t* n_out);
BH_API int bh_check_invariants(bh_heap* heap, int* ok, char* detail,   /* check_invariants() heap.cpp:726-770 */
                               size_t detail_cap);
/* Raw layout (slot order, slot 1 first) + partial buffer; for parity tests. */
BH_API int bh_dump(bh_heap* heap, void* keys_out, uint64_t keys_cap, void* partial_out,
                   uint32_t* partial_len, uint32_t* states_out);
BH_API int bh_info(bh_heap* heap, uint32_t* k, uint32_t* key_bits, uint64_t* slot_count,
                   uint32_t* max_nodes, int* variant, uint32_t* threads_per_cta,
                   uint32_t* max_ctas);

/* Device event log (BH_FLAG_RECORD handles).  Each event: ts (global device
 * clock), op index, kind (0 inv, 1 res, 2 lock acquired, 3 lock released,
 * 4 lock acquired on the refill source -- the last node a delete moves into
 * the root, held only to copy and blank it, never across a wait), node slot.  Mirrors Recorder::op_begin/lock_acquired/lock_released/op_end
 * (proj/include/batchheap/instrumentation.hpp:20-57). Returns the number of
 * events of the last bulk run (events sorted by op, then ts). */
typedef struct {
    uint64_t ts;
    uint32_t op;
    uint16_t kind;
    uint16_t pad;
    uint64_t node;
} bh_event;
BH_API int bh_history(bh_heap* heap, bh_event* out, uint64_t cap, uint64_t* n_out);

/* Cycle profile of BH_FLAG_PROFILE handles (no reference analogue; the
 * reference's only timing is wall clock around whole runs).  Fills up to
 * `cap` words: [0] insert ops, [1] sort cycles, [2] root-wait cycles,
 * [3] root-hold cycles, [4] post-root cycles, [5] delete ops, [6] delete
 * root-wait, [7] delete root-hold, [8] delete heapify cycles, [9] child-lock
 * wait cycles, [10] heapify levels, [11] CTA busy cycles.  reset != 0 zeroes
 * the counters after reading. */
BH_API int bh_profile(bh_heap* heap, uint64_t* out, uint32_t cap, int reset);

/* Thread-local message for the last failing call on this thread. */
BH_API const char* bh_last_error(void);

/* ---------------------------------------------------------------------------
 * Batch primitives (reference batch_core) as standalone device kernels over
 * DEVICE buffers, exposed for parity tests and reuse.
 * ------------------------------------------------------------------------- */
/* sort_batch (proj/src/batch.cpp:7-19): sorts `batches` rows of `lens[i]`
 * keys (stride k) in place; row tails past len are set to the sentinel. */
BH_API int bh_sort_batches(uint32_t key_bits, uint32_t k, void* keys, const uint32_t* lens,
                           uint64_t batches, void* stream);
/* merge_and_sort (proj/src/batch.cpp:32-42) on full rows: for each pair i,
 * hi[i] = k smallest of a[i] U b[i], lo[i] = the rest (ties take a first). */
BH_API int bh_merge_split(uint32_t key_bits, uint32_t k, const void* a, const void* b, void* hi,
                          void* lo, uint64_t pairs, void* stream);

/* Bit-reversal target selection (proj/include/batchheap/bitrev.hpp:15-42). */
BH_API uint64_t bh_slot_for_rank(uint64_t rank);
BH_API uint64_t bh_bit_reverse(uint64_t x, unsigned bits);

/* Workload key generator (generate_keys, proj/src/workload.cpp:162-180):
 * order 0 random (mt19937_64, uniform [0, 2^32-1]), 1 ascend, 2 descend.
 * Writes 64-bit keys, or 32-bit when key_bits == 32. */
BH_API int bh_generate_keys(int order, uint64_t n, uint64_t seed, uint32_t key_bits, void* out);

/* ---------------------------------------------------------------------------
 * Application drivers: the reference's SSSP and knapsack
 * branch-and-bound on the device heap.  Host buffers in and out; every
 * per-node step (heap ops, relaxation, child expansion) runs on `device`.
 * ------------------------------------------------------------------------- */
/* grid_graph(rows, cols, seed) (proj/src/graph.cpp:174-193) in the CSR layout
 * of Graph::Graph (graph.cpp:12-30): offsets[rows*cols+1], and per arc the
 * target node and weight (uniform [1,1000] from mt19937_64(seed)). */
BH_API uint64_t bh_grid_graph_edges(uint32_t rows, uint32_t cols);
BH_API int bh_grid_graph(uint32_t rows, uint32_t cols, uint64_t seed, uint64_t* offsets,
                         uint32_t* adj_node, uint32_t* adj_weight);

/* SsspConfig (proj/include/batchheap/sssp.hpp:27-31); the reference's host
 * workers become the heap's persistent CTAs (0 = all co-resident). */
typedef struct {
    uint64_t threshold;          /* active-set size that engages the heap (0 -> 10000) */
    uint32_t heap_node_capacity; /* k (0 -> 1024; the reference uses 32) */
    uint32_t ctas;
    uint64_t reserved;
} bh_sssp_cfg;
typedef struct {
    uint64_t visits;            /* SsspResult::visits: non-stale explorations */
    uint64_t rounds;
    uint64_t keys_through_heap; /* keys funnelled through the heap */
    double seconds;
} bh_sssp_stats;
/* sssp(graph, source, config) (proj/src/sssp.cpp:118-194).  dist: n_nodes
 * distances, UINT64_MAX where unreachable; BH_E_INVALID_KEY when a distance
 * exceeds the key encoding (sssp.cpp:16-20 overflow_error). */
BH_API int bh_sssp(uint32_t n_nodes, const uint64_t* offsets, const uint32_t* adj_node,
                   const uint32_t* adj_weight, uint32_t source, const bh_sssp_cfg* cfg, int device,
                   uint64_t* dist, bh_sssp_stats* stats);

/* KnapsackType (proj/include/batchheap/knapsack.hpp:16-21). */
enum {
    BH_KS_STRONGLY_CORRELATED = 0,
    BH_KS_ALMOST_STRONGLY_CORRELATED = 1,
    BH_KS_EVEN_ODD = 2,
    BH_KS_SUBSET_SUM = 3
};
/* generate_knapsack(type, n, range, seed) (proj/src/knapsack.cpp:22-66):
 * fills weight[n], benefit[n]; returns the capacity (0 on bad arguments). */
BH_API uint64_t bh_generate_knapsack(int type, uint32_t n, uint32_t range, uint64_t seed,
                                     uint32_t* weight, uint32_t* benefit);
/* BbConfig (knapsack.hpp:56-60) plus the device round shape. */
typedef struct {
    uint64_t gc_threshold;       /* keys; 0 disables GC (reference 1 << 16) */
    uint32_t heap_node_capacity; /* k (0 -> 1024; the reference uses 32) */
    uint32_t ctas;               /* persistent CTAs (0 = all co-resident) */
    uint32_t pop_ops;            /* deleteMin batches per round (0 -> 4) */
    uint32_t reserved;
    uint64_t arena_nodes;        /* node slots (recycled; 0 -> 1 << 28) */
    uint64_t max_explored;       /* node budget: BH_E_CAPACITY past it (0 -> 1 << 29) */
} bh_bb_cfg;
/* BbOutcome (knapsack.hpp:62-66) plus round statistics. */
typedef struct {
    uint64_t best;
    uint64_t explored;
    uint64_t gc_passes;
    uint64_t rounds;
    uint64_t arena_nodes;
    double seconds;
} bh_bb_outcome;
/* knapsack_bb(instance, config) (proj/src/knapsack.cpp:206-368): the
 * optimum of the 0/1 knapsack; BH_E_CAPACITY when the node slots or the
 * node budget run out (the reference's "branch-and-bound arena exhausted",
 * which it raises inside a worker and terminates on). */
BH_API int bh_knapsack_bb(uint32_t n, const uint32_t* weight, const uint32_t* benefit, uint64_t capacity,
                          const bh_bb_cfg* cfg, int device, bh_bb_outcome* out);

/* plan_batches (proj/src/bench.cpp:21-47): the batch lengths the reference's
 * benchmark inserts for n_keys keys split over `workers` contiguous shares
 * (full_batch_pct % full k-batches, the rest 1..k-1 keys, mt19937_64 per
 * worker).  Writes up to cap lengths (and each batch's worker) in worker
 * order; *n_out = number of batches.  Pass lens = NULL to size. */
BH_API int bh_plan_batches(uint32_t k, uint64_t n_keys, uint32_t workers, uint32_t full_batch_pct,
                           uint64_t seed, uint32_t* lens, uint32_t* worker_of, uint64_t cap,
                           uint64_t* n_out);

/* Library build identity (sm arch, compile flags). */
BH_API const char* bh_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* BATCHHEAP_B200_H */

// batchheap_b200.hpp -- C++ facade with the reference's class shape.
//
// Rebuilds batchheap::GeneralizedHeap (reference
// proj/include/batchheap/heap.hpp:72-181) on top of the C ABI in
// batchheap_b200.h, so reference callers (proj/src/bench.cpp,
// proj/src/sssp.cpp, proj/src/knapsack.cpp, proj/tests/test_heap.cpp) port
// by changing the include and namespace: same constructor arguments, same
// methods, same exception types, Key = uint64_t.  Every call runs on the GPU.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "batchheap_b200.h"

namespace batchheap_b200 {

using Key = std::uint64_t;  // proj/include/batchheap/batch.hpp:17
inline constexpr Key kMaxKey = ~Key{0};

struct ConfigError : std::runtime_error {  // batch.hpp:23-25
    using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {  // batch.hpp:26-28
    using std::runtime_error::runtime_error;
};
struct EmptyHeapError : std::runtime_error {  // batch.hpp:29-31
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class Variant : std::uint8_t { TD = BH_TD, BU = BH_BU };  // history.hpp:23

struct HeapOptions {  // heap.hpp:43-47
    bool elide_merges = true;
};

using HeapCounters = bh_counters;  // heap.hpp:49-58, same field names
using HeapPeek = bh_peek;          // heap.hpp:60-65

struct InvariantReport {  // heap.hpp:67-70
    bool ok = true;
    std::string detail;
};

namespace detail {
inline void check(int rc) {
    if (rc == BH_OK) return;
    const std::string msg = bh_last_error();
    switch (rc) {
        case BH_E_CONFIG: throw ConfigError(msg);
        case BH_E_CAPACITY: throw CapacityError(msg);
        case BH_E_EMPTY: throw EmptyHeapError(msg);
        case BH_E_INVALID_KEY: throw std::invalid_argument(msg);
        case BH_E_CUDA: throw DeviceError(msg);
        default: throw std::logic_error(msg);
    }
}
}  // namespace detail

class GeneralizedHeap {
  public:
    // heap.hpp:74-75 (the Recorder* argument becomes `record`: the device
    // event log read back with history()).
    GeneralizedHeap(Variant variant, std::uint32_t k, std::uint32_t max_nodes,
                    HeapOptions options = {}, bool record = false, int device = 0)
        : variant_(variant), k_(k), max_nodes_(max_nodes) {
        const std::uint32_t flags = (options.elide_merges ? BH_FLAG_ELIDE_MERGES : 0u) |
                                    (record ? BH_FLAG_RECORD : 0u);
        detail::check(bh_create(&h_, static_cast<int>(variant), k, max_nodes, 64, flags, device));
    }
    ~GeneralizedHeap() { bh_destroy(h_); }
    GeneralizedHeap(const GeneralizedHeap&) = delete;
    GeneralizedHeap& operator=(const GeneralizedHeap&) = delete;

    // heap.hpp:81-83
    void insert(std::span<const Key> items) {
        detail::check(bh_insert(h_, items.data(), static_cast<std::uint32_t>(items.size())));
    }

    // heap.hpp:86
    std::vector<Key> delete_min() {
        auto r = try_delete_min();
        if (!r) throw EmptyHeapError("delete_min: heap empty");
        return std::move(*r);
    }

    // heap.hpp:88
    std::optional<std::vector<Key>> try_delete_min() {
        std::vector<Key> out(k_);
        std::uint32_t n = 0;
        const int rc = bh_delete_min(h_, out.data(), &n);
        if (rc == BH_E_EMPTY) return std::nullopt;
        detail::check(rc);
        out.resize(n);
        return out;
    }

    // Bulk path: ops execute concurrently in one persistent-kernel launch.
    void run_ops(std::span<const bh_op> ops, std::span<const Key> key_pool, std::span<Key> out_pool,
                 std::uint32_t* out_status = nullptr, std::uint32_t* out_lens = nullptr,
                 std::uint64_t* out_seq = nullptr, std::uint32_t ctas = 0) {
        bh_run_cfg cfg{ctas, 0, nullptr};
        detail::check(bh_run_ops(h_, ops.data(), ops.size(), key_pool.data(), key_pool.size(),
                                 out_pool.data(), out_pool.size(), out_status, out_lens, out_seq, &cfg));
    }

    HeapPeek peek_stats() const {  // heap.hpp:90
        HeapPeek p{};
        detail::check(bh_peek_stats(h_, &p));
        return p;
    }
    HeapCounters counters() const {  // heap.hpp:91
        HeapCounters c{};
        detail::check(bh_get_counters(h_, &c));
        return c;
    }
    void reset_counters() { detail::check(bh_reset_counters(h_)); }  // heap.hpp:92

    Variant variant() const { return variant_; }
    std::uint32_t node_capacity() const { return k_; }
    std::uint32_t max_nodes() const { return max_nodes_; }

    std::uint64_t select_insert_target() const {  // heap.hpp:99
        std::uint64_t slot = 0;
        detail::check(bh_select_insert_target(h_, &slot));
        return slot;
    }

    std::vector<Key> collect_resident() const {  // heap.hpp:102
        std::uint64_t n = 0;
        detail::check(bh_collect_resident(h_, nullptr, 0, &n));
        std::vector<Key> out(n);
        detail::check(bh_collect_resident(h_, out.data(), out.size(), &n));
        return out;
    }

    InvariantReport check_invariants() const {  // heap.hpp:104
        int ok = 0;
        char buf[4096];
        detail::check(bh_check_invariants(h_, &ok, buf, sizeof(buf)));
        return {ok != 0, buf};
    }

    std::vector<bh_event> history() const {
        std::uint64_t n = 0;
        detail::check(bh_history(h_, nullptr, 0, &n));
        std::vector<bh_event> ev(n);
        detail::check(bh_history(h_, ev.data(), ev.size(), &n));
        return ev;
    }

    bh_heap* handle() const { return h_; }

  private:
    bh_heap* h_ = nullptr;
    Variant variant_;
    std::uint32_t k_;
    std::uint32_t max_nodes_;
};

// ---- drivers (proj/include/batchheap/{graph,sssp,knapsack}.hpp) --------
inline constexpr std::uint64_t kUnreachable = ~std::uint64_t{0};  // sssp.hpp:18-19

struct Graph {  // graph.hpp:26-50, CSR
    std::vector<std::uint64_t> offsets;
    std::vector<std::uint32_t> nbr;
    std::vector<std::uint32_t> weight;
    std::uint32_t node_count() const { return static_cast<std::uint32_t>(offsets.size() - 1); }
    std::uint64_t edge_count() const { return nbr.size(); }
};

inline Graph grid_graph(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed) {  // graph.cpp:174-193
    Graph g;
    const std::uint64_t m = bh_grid_graph_edges(rows, cols);
    g.offsets.resize(std::uint64_t{rows} * cols + 1);
    g.nbr.resize(m);
    g.weight.resize(m);
    detail::check(bh_grid_graph(rows, cols, seed, g.offsets.data(), g.nbr.data(), g.weight.data()));
    return g;
}

struct SsspConfig {  // sssp.hpp:27-31 (workers -> persistent CTAs; k default 1024 on the device)
    std::uint64_t threshold = 10'000;
    std::uint32_t ctas = 0;
    std::uint32_t heap_node_capacity = 1024;
};

struct SsspResult {  // sssp.hpp:21-24
    std::vector<std::uint64_t> dist;
    std::uint64_t visits = 0;
};

inline SsspResult sssp(const Graph& g, std::uint32_t source, const SsspConfig& config = {}, int device = 0) {
    SsspResult r;
    r.dist.resize(g.node_count());
    bh_sssp_cfg c{config.threshold, config.heap_node_capacity, config.ctas, 0};
    bh_sssp_stats st{};
    detail::check(bh_sssp(g.node_count(), g.offsets.data(), g.nbr.data(), g.weight.data(), source, &c, device,
                          r.dist.data(), &st));
    r.visits = st.visits;
    return r;
}

enum class KnapsackType { StronglyCorrelated, AlmostStronglyCorrelated, EvenOdd, SubsetSum };  // knapsack.hpp:16

struct KnapsackInstance {  // knapsack.hpp:23-31
    KnapsackType type = KnapsackType::SubsetSum;
    std::uint32_t n = 0;
    std::uint32_t range = 0;
    std::vector<std::uint32_t> weight;
    std::vector<std::uint32_t> benefit;
    std::uint64_t capacity = 0;
};

inline KnapsackInstance generate_knapsack(KnapsackType type, std::uint32_t n, std::uint32_t range,
                                          std::uint64_t seed) {  // knapsack.cpp:22-66
    KnapsackInstance inst;
    inst.type = type;
    inst.n = n;
    inst.range = range;
    inst.weight.resize(n);
    inst.benefit.resize(n);
    inst.capacity =
        bh_generate_knapsack(static_cast<int>(type), n, range, seed, inst.weight.data(), inst.benefit.data());
    if (inst.capacity == 0) detail::check(BH_E_CONFIG);
    return inst;
}

struct BbConfig {  // knapsack.hpp:56-60 (device defaults: k 1024, GC at 2^20)
    std::uint32_t ctas = 0;
    std::uint64_t gc_threshold = 1 << 20;
    std::uint32_t heap_node_capacity = 1024;
    std::uint32_t pop_ops = 4;
};

struct BbOutcome {  // knapsack.hpp:62-66
    std::uint64_t best = 0;
    std::uint64_t explored = 0;
    std::uint64_t gc_passes = 0;
};

inline BbOutcome knapsack_bb(const KnapsackInstance& inst, const BbConfig& config = {}, int device = 0) {
    bh_bb_cfg c{config.gc_threshold, config.heap_node_capacity, config.ctas, config.pop_ops, 0, 0, 0};
    bh_bb_outcome o{};
    detail::check(bh_knapsack_bb(inst.n, inst.weight.data(), inst.benefit.data(), inst.capacity, &c, device, &o));
    return {o.best, o.explored, o.gc_passes};
}

// Bit-reversal target selection (proj/include/batchheap/bitrev.hpp).
inline std::uint64_t slot_for_rank(std::uint64_t rank) { return bh_slot_for_rank(rank); }
inline std::uint64_t bit_reverse(std::uint64_t x, unsigned bits) { return bh_bit_reverse(x, bits); }

}  // namespace batchheap_b200

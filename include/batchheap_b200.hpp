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

// Bit-reversal target selection (proj/include/batchheap/bitrev.hpp).
inline std::uint64_t slot_for_rank(std::uint64_t rank) { return bh_slot_for_rank(rank); }
inline std::uint64_t bit_reverse(std::uint64_t x, unsigned bits) { return bh_bit_reverse(x, bits); }

}  // namespace batchheap_b200

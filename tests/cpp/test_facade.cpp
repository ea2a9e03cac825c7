// C++ facade parity: reference test cases (proj/tests/test_heap.cpp) run
// unchanged in shape through batchheap_b200::GeneralizedHeap.  Built by
// tests/test_cpp_facade.py; exits non-zero on the first failed check.
#include <algorithm>
#include <queue>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>

#include "batchheap_b200.hpp"

using namespace batchheap_b200;

static int failures = 0;
#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                 \
        }                                                               \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::vector<Key> random_keys(std::mt19937_64& rng, std::size_t n, Key range = 1'000'000) {
    std::uniform_int_distribution<Key> dist(0, range);
    std::vector<Key> keys(n);
    for (auto& k : keys) k = dist(rng);
    return keys;
}

int main() {
    {  // construction (test_heap.cpp:23-33)
        GeneralizedHeap heap(Variant::TD, 4, 1024);
        CHECK(heap.peek_stats().key_count == 0);
        CHECK(throws<ConfigError>([] { GeneralizedHeap(Variant::TD, 3, 8); }));
        CHECK(throws<ConfigError>([] { GeneralizedHeap(Variant::TD, 4, 0); }));
    }
    {  // partial insert merges through root, property 3 (:41-51)
        GeneralizedHeap heap(Variant::TD, 2, 16);
        heap.insert(std::vector<Key>{5, 1});
        heap.insert(std::vector<Key>{3});
        CHECK(heap.peek_stats().node_count == 1);
        CHECK(heap.peek_stats().partial_len == 1);
        CHECK(heap.check_invariants().ok);
        CHECK((heap.delete_min() == std::vector<Key>{1, 3}));
        CHECK((heap.delete_min() == std::vector<Key>{5}));
        CHECK(throws<EmptyHeapError>([&] { heap.delete_min(); }));
        CHECK(!heap.try_delete_min().has_value());
    }
    for (Variant v : {Variant::TD, Variant::BU}) {  // heapsort oracle (:89-108)
        GeneralizedHeap heap(v, 4, 1024);
        std::mt19937_64 rng(1234);
        auto keys = random_keys(rng, 1024);
        for (std::size_t at = 0; at < keys.size(); at += 4)
            heap.insert(std::span<const Key>(keys).subspan(at, 4));
        std::vector<Key> drained;
        for (int i = 0; i < 256; ++i) {
            auto b = heap.delete_min();
            drained.insert(drained.end(), b.begin(), b.end());
        }
        std::sort(keys.begin(), keys.end());
        CHECK(drained == keys);
    }
    {  // capacity error before mutation (:159-170)
        GeneralizedHeap heap(Variant::TD, 2, 2);
        heap.insert(std::vector<Key>{1, 2});
        heap.insert(std::vector<Key>{3, 4});
        auto before = heap.collect_resident();
        CHECK(throws<CapacityError>([&] { heap.insert(std::vector<Key>{5, 6}); }));
        CHECK(heap.collect_resident() == before);
        heap.insert(std::vector<Key>{9});
        CHECK(heap.peek_stats().key_count == 5);
        CHECK(throws<CapacityError>([&] { heap.select_insert_target(); }));
        CHECK(throws<std::invalid_argument>([&] { heap.insert(std::vector<Key>{kMaxKey}); }));
    }
    for (Variant v : {Variant::TD, Variant::BU}) {  // concurrent callers (test_stress.cpp shape)
        GeneralizedHeap heap(v, 8, 8 * 400 + 8);
        std::vector<std::vector<Key>> ins(8), del(8);
        std::vector<std::thread> th;
        for (int w = 0; w < 8; ++w)
            th.emplace_back([&, w] {
                std::mt19937_64 rng(w + 17);
                for (int i = 0; i < 300; ++i) {
                    if (rng() & 1) {
                        auto keys = random_keys(rng, 1 + rng() % 8, 1 << 20);
                        heap.insert(keys);
                        ins[w].insert(ins[w].end(), keys.begin(), keys.end());
                    } else if (auto r = heap.try_delete_min()) {
                        del[w].insert(del[w].end(), r->begin(), r->end());
                    }
                }
            });
        for (auto& t : th) t.join();
        CHECK(heap.check_invariants().ok);
        std::vector<Key> a, b = heap.collect_resident();
        for (int w = 0; w < 8; ++w) {
            a.insert(a.end(), ins[w].begin(), ins[w].end());
            b.insert(b.end(), del[w].begin(), del[w].end());
        }
        std::sort(a.begin(), a.end());
        std::sort(b.begin(), b.end());
        CHECK(a == b);
    }
    {  // bit-reversal targets (:146-157)
        GeneralizedHeap heap(Variant::TD, 2, 16);
        CHECK(heap.select_insert_target() == 1);
        const std::uint64_t expect[] = {2, 3, 4, 6};
        for (int i = 0; i < 4; ++i) {
            heap.insert(std::vector<Key>{Key(2 * i + 1), Key(2 * i + 2)});
            CHECK(heap.select_insert_target() == expect[i]);
        }
    }
    {  // drivers in the reference's call shape (batchheap_main.cpp:192, :239-246):
       // SSSP vs a textbook Dijkstra, B&B vs the DP optimum
        const Graph g = grid_graph(40, 30, 3);
        auto r = sssp(g, 7, SsspConfig{64, 0, 32});
        std::vector<std::uint64_t> d(g.node_count(), kUnreachable);
        using Item = std::pair<std::uint64_t, std::uint32_t>;
        std::priority_queue<Item, std::vector<Item>, std::greater<>> q;
        d[7] = 0;
        q.push({0, 7});
        while (!q.empty()) {
            auto [du, u] = q.top();
            q.pop();
            if (du != d[u]) continue;
            for (std::uint64_t a = g.offsets[u]; a < g.offsets[u + 1]; ++a) {
                const std::uint64_t c = du + g.weight[a];
                if (c < d[g.nbr[a]]) {
                    d[g.nbr[a]] = c;
                    q.push({c, g.nbr[a]});
                }
            }
        }
        CHECK(r.dist == d);
        CHECK(throws<ConfigError>([&] { sssp(g, g.node_count()); }));
        for (auto t : {KnapsackType::StronglyCorrelated, KnapsackType::SubsetSum}) {
            const auto inst = generate_knapsack(t, 40, 1000, 5);
            std::vector<std::uint64_t> table(inst.capacity + 1, 0);
            for (std::uint32_t i = 0; i < inst.n; ++i)
                for (std::uint64_t c = inst.capacity; c >= inst.weight[i]; --c)
                    table[c] = std::max(table[c], table[c - inst.weight[i]] + inst.benefit[i]);
            CHECK(knapsack_bb(inst).best == table[inst.capacity]);
        }
    }
    std::printf("facade: %d failures\n", failures);
    return failures ? 1 : 0;
}

// ref_harness.cpp -- TEST / BASELINE INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference library compiled from
// /root/reference/proj/src (oracle/Makefile -> oracle/_ref/libbatchheap_ref.so).
// Used by tests/ to pin the oracle and the CUDA path against the reference
// itself, and by bench.py's cpu_baseline / --impl reference legs to time the
// reference's own CPU implementation.  Never linked by the product.
//
// ref_phase() is the phase-split timer of SURVEY.md Appendix A step 3: W
// threads insert batches b = w (mod W) into GeneralizedHeap(v, K, N/K+W+2),
// barrier, then every thread calls try_delete_min until `remaining` reaches
// zero (the loop shape of proj/src/bench.cpp:81-101); steady_clock per phase,
// key generation excluded (proj/src/bench.cpp:117-124).
#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <memory>
#include <random>
#include <span>
#include <thread>
#include <vector>

#include "batchheap/bench.hpp"
#include "batchheap/graph.hpp"
#include "batchheap/heap.hpp"
#include "batchheap/knapsack.hpp"
#include "batchheap/lincheck.hpp"
#include "batchheap/seq_heap.hpp"
#include "batchheap/sssp.hpp"
#include "batchheap/workload.hpp"

using namespace batchheap;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return 2;
    } catch (const EmptyHeapError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_generate_keys(int order, std::uint64_t n, std::uint64_t seed, std::uint64_t* out) {
    auto keys = generate_keys(static_cast<KeyOrder>(order), n, seed);
    std::memcpy(out, keys.data(), n * sizeof(std::uint64_t));
}

// ---------------------------------------------------------------- heap ----
void* ref_heap_create(int variant, std::uint32_t k, std::uint32_t max_nodes, int elide) {
    GeneralizedHeap* h = nullptr;
    HeapOptions opt;
    opt.elide_merges = elide != 0;
    if (guarded([&] { h = new GeneralizedHeap(variant ? Variant::BU : Variant::TD, k, max_nodes, opt); }))
        return nullptr;
    return h;
}
void ref_heap_destroy(void* h) { delete static_cast<GeneralizedHeap*>(h); }

int ref_heap_insert(void* h, const std::uint64_t* keys, std::uint32_t n) {
    return guarded([&] {
        static_cast<GeneralizedHeap*>(h)->insert(std::span<const Key>(keys, n));
    });
}

int ref_heap_delete(void* h, std::uint64_t* out, std::uint32_t* n_out) {
    *n_out = 0;
    return guarded([&] {
        auto r = static_cast<GeneralizedHeap*>(h)->delete_min();
        std::memcpy(out, r.data(), r.size() * sizeof(Key));
        *n_out = static_cast<std::uint32_t>(r.size());
    });
}

void ref_heap_peek(void* h, std::uint64_t* out4) {
    auto p = static_cast<GeneralizedHeap*>(h)->peek_stats();
    out4[0] = p.node_count;
    out4[1] = p.key_count;
    out4[2] = p.partial_len;
    out4[3] = p.level_count;
}

void ref_heap_counters(void* h, std::uint64_t* out8) {
    auto c = static_cast<GeneralizedHeap*>(h)->counters();
    std::uint64_t v[8] = {c.inserts, c.deletes, c.merges, c.elided_merges,
                          c.early_stops, c.propagation_node_visits, c.coop_handoffs,
                          c.max_partial_len};
    std::memcpy(out8, v, sizeof(v));
}

std::uint64_t ref_heap_collect(void* h, std::uint64_t* out, std::uint64_t cap) {
    auto keys = static_cast<GeneralizedHeap*>(h)->collect_resident();
    std::memcpy(out, keys.data(), std::min<std::uint64_t>(cap, keys.size()) * sizeof(Key));
    return keys.size();
}

int ref_heap_check(void* h) { return static_cast<GeneralizedHeap*>(h)->check_invariants().ok ? 1 : 0; }

// --------------------------------------------------------- phase timer ----
// Returns 0 on success; times[0]=insert s, times[1]=delete s. verify=1
// checks that the delete stream equals the sorted input (W=1 order) or the
// multiset (W>1), returning 6 on mismatch.
int ref_phase(int variant, std::uint32_t k, std::uint64_t n_keys, std::uint32_t workers,
              std::uint64_t seed, int verify, double* times) {
    return guarded([&] {
        std::vector<Key> keys = generate_keys(KeyOrder::Random, n_keys, seed);
        const std::uint64_t max_nodes = n_keys / k + workers + 2;
        GeneralizedHeap heap(variant ? Variant::BU : Variant::TD, k,
                             static_cast<std::uint32_t>(max_nodes));
        const std::uint64_t batches = (n_keys + k - 1) / k;
        std::atomic<std::uint64_t> remaining{n_keys};
        std::vector<std::vector<Key>> deleted(workers);
        std::barrier sync(workers + 1);
        std::vector<std::thread> threads;
        for (std::uint32_t w = 0; w < workers; ++w) {
            threads.emplace_back([&, w] {
                sync.arrive_and_wait();
                for (std::uint64_t b = w; b < batches; b += workers) {
                    const std::uint64_t at = b * k;
                    heap.insert(std::span<const Key>(keys).subspan(
                        at, std::min<std::uint64_t>(k, n_keys - at)));
                }
                sync.arrive_and_wait();
                sync.arrive_and_wait();
                while (remaining.load(std::memory_order_relaxed) != 0) {
                    auto r = heap.try_delete_min();
                    if (!r) {
                        std::this_thread::yield();
                        continue;
                    }
                    remaining.fetch_sub(r->size(), std::memory_order_relaxed);
                    if (verify) deleted[w].insert(deleted[w].end(), r->begin(), r->end());
                }
                sync.arrive_and_wait();
            });
        }
        auto t0 = std::chrono::steady_clock::now();
        sync.arrive_and_wait();
        sync.arrive_and_wait();
        auto t1 = std::chrono::steady_clock::now();
        sync.arrive_and_wait();
        auto t2 = std::chrono::steady_clock::now();
        sync.arrive_and_wait();
        auto t3 = std::chrono::steady_clock::now();
        for (auto& t : threads) t.join();
        times[0] = std::chrono::duration<double>(t1 - t0).count();
        times[1] = std::chrono::duration<double>(t3 - t2).count();
        if (verify) {
            std::vector<Key> all;
            for (auto& d : deleted) all.insert(all.end(), d.begin(), d.end());
            std::sort(keys.begin(), keys.end());
            if (workers == 1) {
                if (all != keys) throw std::runtime_error("drain != sorted input");
            } else {
                std::sort(all.begin(), all.end());
                if (all != keys) throw std::runtime_error("multiset mismatch");
            }
        }
    });
}

// Reference's own sweep row (proj/src/bench.cpp:163-185): correctness pass
// then timed pass; out[0]=wall s, out[1]=ops, out[2]=merges,
// out[3]=early_stops, out[4]=mean_nodes_traversed, out[5]=inserts,
// out[6]=deletes (out must hold 7 doubles).
int ref_run_workload(int variant, std::uint32_t k, std::uint32_t workers, std::uint64_t total_keys,
                     int order, int pattern, std::uint32_t initial_levels,
                     std::uint32_t full_pct, std::uint64_t seed, double* out) {
    return guarded([&] {
        WorkloadSpec s;
        s.variant = variant ? Variant::BU : Variant::TD;
        s.k = k;
        s.workers = workers;
        s.total_keys = total_keys;
        s.key_order = static_cast<KeyOrder>(order);
        s.op_pattern = static_cast<OpPattern>(pattern);
        s.initial_levels = initial_levels;
        s.full_batch_pct = full_pct;
        s.seed = seed;
        BenchRow row = run_workload(s);
        out[0] = row.wall_seconds;
        out[1] = static_cast<double>(row.ops);
        out[2] = static_cast<double>(row.counters.merges);
        out[3] = static_cast<double>(row.counters.early_stops);
        out[4] = row.mean_nodes_traversed;
        out[5] = static_cast<double>(row.counters.inserts);
        out[6] = static_cast<double>(row.counters.deletes);
    });
}

// The reference's own concurrent stress runner (proj/src/workload.cpp:75-147)
// plus its checkers (proj/src/lincheck.cpp).  out[0] invariants ok,
// out[1] multiset ok, out[2] constructive check (check_td / check_bu) ok,
// out[3] mutual exclusion ok, out[4] lock order ok, out[5] ops recorded.
int ref_stress(int variant, std::uint32_t k, std::uint32_t workers, std::uint64_t ops_per_worker,
               std::uint32_t partial_pct, std::uint64_t seed, std::uint64_t key_range, int elide,
               int* out) {
    return guarded([&] {
        StressSpec s;
        s.variant = variant ? Variant::BU : Variant::TD;
        s.k = k;
        s.workers = workers;
        s.ops_per_worker = ops_per_worker;
        s.partial_pct = partial_pct;
        s.seed = seed;
        s.key_range = key_range;
        s.options.elide_merges = elide != 0;
        s.watchdog_seconds = 60;
        StressOutcome o = run_stress(s);
        out[0] = o.invariants.ok;
        out[1] = o.multiset_ok;
        out[2] = (variant ? check_bu(o.history) : check_td(o.history)).pass;
        out[3] = check_mutual_exclusion(o.history).ok;
        out[4] = check_lock_order(o.history).ok;
        out[5] = static_cast<int>(o.history.ops.size());
    });
}

// ---------------------------------------------------------- apps ----------
// grid_graph + dijkstra: writes distances for `source`.
int ref_grid_dijkstra(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed,
                      std::uint32_t source, std::uint64_t* dist) {
    return guarded([&] {
        Graph g = grid_graph(rows, cols, seed);
        auto d = dijkstra(g, source);
        std::memcpy(dist, d.data(), d.size() * sizeof(std::uint64_t));
    });
}

// The reference's heap-driven SSSP (proj/src/sssp.cpp:118-194).
int ref_grid_sssp(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed, std::uint32_t source,
                  std::uint64_t threshold, std::uint32_t workers, std::uint64_t* dist,
                  std::uint64_t* visits, double* seconds) {
    return guarded([&] {
        Graph g = grid_graph(rows, cols, seed);
        SsspConfig cfg;
        cfg.threshold = threshold;
        cfg.workers = workers;
        auto t0 = std::chrono::steady_clock::now();
        auto r = sssp(g, source, cfg);
        auto t1 = std::chrono::steady_clock::now();
        std::memcpy(dist, r.dist.data(), r.dist.size() * sizeof(std::uint64_t));
        *visits = r.visits;
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

std::uint64_t ref_generate_knapsack(int type, std::uint32_t n, std::uint32_t range,
                                    std::uint64_t seed, std::uint32_t* w, std::uint32_t* b) {
    auto inst = generate_knapsack(static_cast<KnapsackType>(type), n, range, seed);
    std::memcpy(w, inst.weight.data(), n * sizeof(std::uint32_t));
    std::memcpy(b, inst.benefit.data(), n * sizeof(std::uint32_t));
    return inst.capacity;
}

std::uint64_t ref_knapsack_dp(int type, std::uint32_t n, std::uint32_t range, std::uint64_t seed) {
    return knapsack_dp(generate_knapsack(static_cast<KnapsackType>(type), n, range, seed));
}

// The reference's branch-and-bound (proj/src/knapsack.cpp:206-368).  An
// arena exhaustion inside a worker thread calls std::terminate in the
// reference: callers run this in a child process.  out3 = best, explored,
// gc passes.
int ref_knapsack_bb(int type, std::uint32_t n, std::uint32_t range, std::uint64_t seed, std::uint32_t workers,
                    std::uint64_t gc_threshold, std::uint32_t k, std::uint64_t* out3, double* seconds) {
    return guarded([&] {
        auto inst = generate_knapsack(static_cast<KnapsackType>(type), n, range, seed);
        BbConfig cfg;
        cfg.workers = workers;
        cfg.gc_threshold = gc_threshold;
        cfg.heap_node_capacity = k;
        auto t0 = std::chrono::steady_clock::now();
        auto o = knapsack_bb(inst, cfg);
        auto t1 = std::chrono::steady_clock::now();
        out3[0] = o.best;
        out3[1] = o.explored;
        out3[2] = o.gc_passes;
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

}  // extern "C"

// bh_internal.h -- layouts shared by the host C ABI and the device kernels.
#pragma once

#include <cstdint>

#include "batchheap_b200.h"

namespace bh {

// Node state words (reference proj/include/batchheap/heap.hpp:107-114).
enum : uint32_t {
    kAvail = 0,
    kInUse = 1,
    kTarget = 2,
    kMarked = 3,
    kInsHold = 4,
    kDelMod = 5,
};

// One state word per 32-byte sector so lock traffic on neighbouring nodes
// never shares an L2 atomic sector.
constexpr uint32_t kStateStride = 8;  // uint32 words
// Root queue lock: one flag per waiter slot, each on its own 128-byte line.
constexpr uint32_t kRootQueue = 4096;
constexpr uint32_t kRootFlagStride = 32;  // uint32 words
// Profile buffer: 48 counters + 4 debug words per CTA (up to 4096 CTAs).
// profile words: counters (64), per-CTA wait notes (4 x 4096), then a
// per-op event timeline of a three-level server (kTlOps ops x 32 clocks)
constexpr uint32_t kTlBase = 64 + 4 * 4096, kTlFirst = 1000, kTlOps = 64;
// per-level BU climb profile (profiling handles): climb steps, parent-claim
// cycles and claim-to-release cycles, indexed by the parent's level
constexpr uint32_t kLvBase = kTlBase + kTlOps * 32, kLvLevels = 32;
constexpr uint32_t kProfWords = kLvBase + 3 * kLvLevels;

// Debug-only protocol toggles (bh_create flags, not in the public header).
constexpr uint32_t kDbgSeqRefill = 0x100;       // reference refill order in every delete
constexpr uint32_t kDbgWriteUnderRoot = 0x200;  // BU target written before the root release
constexpr uint32_t kDbgSerialLanes = 0x400;     // claim children one after the other
constexpr uint32_t kDbgNoCombine = 0x800;       // no insert combining in the root queue lock
constexpr uint32_t kDbgParkClimb = 0x1000;      // reference BU climb (fenced park, reload on re-take)
constexpr uint32_t kDbgNoDelServe = 0x2000;     // no delete serving in the root queue lock
constexpr uint32_t kDbgNoGate = 0x8000;         // measurement only: BU phase gate off (the reference's race returns)
constexpr uint32_t kDbgServe3 = 0x4000;         // three-level delete server (experimental, DESIGN.md s.6): SERVE3=1 builds, where it fits

// Heap header, root-lock guarded (reference heap.hpp:173-177).  One cache
// line; the partial buffer follows in its own allocation.
struct alignas(128) Header {
    unsigned long long node_count;
    unsigned long long insert_count;
    unsigned long long delete_count;  // root-lock sequence of deletes
    unsigned long long root_seq;      // root-lock sequence of all ops
    unsigned long long partial_len;
    unsigned long long error_flags;   // protocol faults seen on device
    unsigned long long clock;         // event-log clock (RECORD)
    unsigned long long pad0[9];
    // second line: waiters' ticket traffic stays off the holder's line
    unsigned long long root_tail;     // root queue-lock ticket dispenser
    unsigned long long climbers;      // BU: in-flight bottom-up climbs
    unsigned long long deleters;      // BU: in-flight delete heapifies
    unsigned long long gate_phase;    // BU: kind that may start (0 climbs, 1 heapifies); root-lock guarded
    unsigned long long gate_closing;  // BU: an op of the other kind waits for the phase
    unsigned long long pad1[11];
};

// Device counters (reference HeapCounters, heap.hpp:49-58).
enum CounterIdx {
    cInserts = 0,
    cDeletes,
    cMerges,
    cElided,
    cEarlyStops,
    cVisits,
    cCoop,
    cMaxPartial,
    cCombined,  // inserts whose root phase a combiner ran (not a reference counter)
    kNumCounters
};

enum ErrorFlag : unsigned long long {
    kErrSentinelEscaped = 1ull << 0,  // heap.cpp:462-463
    kErrInteriorEmpty = 1ull << 1,    // heap.cpp:286 assert
    kErrEventOverflow = 1ull << 2,
    kErrRetake = 1ull << 3,           // gated BU climb: re-take CAS of the parked slot failed
    kErrStuck = 1ull << 4,            // a spin wait passed ~4 s (deadlock watchdog, workload.cpp:22-53)
};

// kEvAcqRefill: acquire of a delete's refill source (refill_root_from,
// heap.cpp:467-531), held only to copy and blank it -- never across a wait --
// so the lock-order check may see it overlap an ancestor's claim (see
// oracle/lincheck.py check_lock_order).
enum EventKind : uint16_t { kEvInv = 0, kEvRes = 1, kEvAcq = 2, kEvRel = 3, kEvAcqRefill = 4 };

struct DevEvent {
    unsigned long long ts;
    uint32_t op;
    uint16_t kind;
    uint16_t pad;
    unsigned long long node;
};

// Everything a kernel needs about one heap (by value as a kernel param).
struct HeapView {
    void* keys;              // slot_count * k keys; node i (1-based) at (i-1)*k
    uint32_t* states;        // (slot_count + 1) * kStateStride
    uint32_t* root_flags;    // kRootQueue * kRootFlagStride
    Header* hdr;
    void* partial;           // k keys
    void* mailbox;           // kRootQueue * k keys: carried batches of served deletes
    unsigned long long* counters;
    unsigned long long* prof;  // non-null on BH_FLAG_PROFILE handles
    unsigned long long slot_count;
    uint32_t k;
    uint32_t max_nodes;
    uint32_t variant;
    uint32_t flags;
};

struct RunView {
    const bh_op* ops;
    unsigned long long n_ops;
    const void* key_pool;
    void* out_pool;
    uint32_t* out_status;
    uint32_t* out_lens;
    unsigned long long* out_seq;
    unsigned long long* ticket;
    DevEvent* events;        // n_ops * ev_per_op (RECORD only)
    uint32_t* event_counts;  // n_ops
    uint32_t ev_per_op;
};

// Kernel launch table entry (one per key width x k).
struct KernelInfo {
    uint32_t threads;
    uint32_t smem_bytes;
    int max_ctas_per_sm;
};

}  // namespace bh

// Sets the thread-local bh_last_error() message (bh_capi.cu); returns code.
extern "C" int bh_internal_fail(int code, const char* msg);

// Device-side dispatch implemented in bh_kernels_*.cu.
extern "C" int bh_internal_launch_ops(uint32_t key_bits, const bh::HeapView* hv, const bh::RunView* rv,
                                      uint32_t ctas, void* stream);
extern "C" int bh_internal_kernel_info(uint32_t key_bits, uint32_t k, bh::KernelInfo* info);
extern "C" int bh_internal_launch_sort(uint32_t key_bits, uint32_t k, void* keys, const uint32_t* lens,
                                       uint64_t batches, void* stream);
extern "C" int bh_internal_launch_merge(uint32_t key_bits, uint32_t k, const void* a, const void* b,
                                        void* hi, void* lo, uint64_t pairs, void* stream);
extern "C" int bh_internal_launch_check(uint32_t key_bits, const bh::HeapView* hv,
                                        unsigned long long* result /* device, 4 words */,
                                        void* stream);
extern "C" int bh_internal_launch_gather(uint32_t key_bits, const bh::HeapView* hv,
                                         unsigned long long nodes, void* out /* device */,
                                         void* stream);
extern "C" int bh_internal_launch_plan(int kind, uint32_t k, uint64_t n_keys, bh_op* ops,
                                       void* stream);

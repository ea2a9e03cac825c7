// bh_heap.cuh -- the concurrent generalized heap as a persistent kernel.
//
// Each CTA repeatedly claims the next operation ticket and executes that whole
// INS or DEL (section 4, "threads in one thread block work together
// for one INS and DEL operation"), following the reference protocol
// (proj/src/heap.cpp) state for state:
//
//   insert      heap.cpp:123-188   root phase: sort, partial buffer, rank
//   insert_td   heap.cpp:218-293   TARGET claim, hand-over-hand merge walk,
//                                  MARKED cooperation (ship_to_root :207-216)
//   insert_bu   heap.cpp:295-407   park/INSHOLD climb, DELMOD skip, early stop
//   do_delete   heap.cpp:420-465   root take, refill (:467-531), partial
//                                  re-merge (:533-545), heapify (:547-667)
//
// The throughput of a lock-based heap is set by chains of dependent lock
// hand-offs and merges, not by bandwidth.  Choices that
// shorten the chains (none changes the protocol's states, transitions, lock
// order or the released node contents):
//   * versioned state words (bh_device.cuh): a node's keys load in the same
//     round trip as the relaxed CAS that claims it (the acquire is the poll
//     that saw the release); both children are claimed by two lanes at once;
//   * the root is a FIFO array queue lock whose holder, when it is a BU
//     full-batch insert, also runs the root phase of the BU full-batch
//     inserts queued behind it (serve_inserts: insert combining), and when
//     it is a BU delete, runs levels 0-1 of the deletes queued behind it from
//     shared memory and hands each one's lower heapify to the next waiter
//     (serve_deletes: delete serving);
//   * heapify_down's two-phase level schedule: the node is released right
//     after the first-half merges that decide its batch; the carried and lo
//     batches are finished afterwards while the other half of the CTA claims
//     the next level and precomputes its H; the root's refill and children
//     claim run side by side;
//   * the gated BU climb (climb_gated): no fence on the park, no reload on
//     the re-take, the carried batch written once;
//   * release fences are paid by a lane whose warp has nothing else to do;
//     the next level's nodes and the next deletes' refill nodes are
//     prefetched into L2; counters are per-CTA registers folded at exit.
//
// Deliberate deviations from the reference, each fixing a reference bug:
//   * heapify's merge elision places the batch holding the smaller keys in
//     the hi child on an equal-maxima tie (heap.cpp:628-636);
//   * BU heaps run a phase gate: a bottom-up climb and a delete heapify
//     never overlap (a phase token, see gate_* below).
#pragma once

#include "bh_device.cuh"
#include "bh_select.cuh"

namespace bh {

static_assert(kStuckFlag == kErrStuck, "watchdog flag bit");

// Releases a delete server has deferred to its next op (kPubLane only).
struct SvPending {
    unsigned long long slot[5];
    unsigned long long op[5];  // op each release belongs to (recorded heaps)
    uint32_t rel[5];
    uint32_t n;
    unsigned long long pub;  // ticket whose hand-off flag is due (0 = none)
    uint32_t pubw;           // its continuation word (slot | release-as-DELMOD << 31)
    unsigned long long pubop;  // op whose continuation it is (recorded heaps)
};

// A served op's record for the control warp of a three-level delete server
// (ring of 4, by the op's index in the hold).
struct Sv3Rec {
    unsigned long long op, off, seq, t, cont;
    unsigned long long relslot[2];
    uint32_t relst[2];
    uint32_t nrel, crel;
    uint32_t rootbuf;  // the op's result: node 1 before the op
    uint32_t c3buf;    // carried batch still to copy into mbox(t + 1) (~0: already there)
    uint32_t cnt_merges, cnt_elided, cnt_early, cnt_visits;
    uint32_t last;     // the hold ends after this op
};

// Shared state of a three-level delete server (serve3): mbarriers between
// its warp roles, the messages they pass, the look-ahead ring.
struct Sv3Shared {
    unsigned long long mb_go[2];   // merge leader -> refill warp g: a refill to run (g = op parity)
    unsigned long long mb_rf[2];   // refill warp g -> merge warps: refill batch in smem
    unsigned long long mb_c3;      // claim warp -> merge warps: level-3 children in smem
    unsigned long long mb_go3;     // merge leader -> claim warp: the op's level-3 claim
    unsigned long long mb_rec;     // merge leader -> control warp: the op's record
    unsigned long long g3_t, g3_op;
    uint32_t g3_hi2, g3_L, g3_R;   // hi2 (0 = leave the loop), destination buffers
    uint32_t g3_j;
    unsigned long long go_last[2]; // refill source rank (0 = leave the loop)
    unsigned long long go_op[2];   // op index (event log)
    uint32_t go_buf[2];            // destination buffer
    uint32_t go_j[2];              // the op's index in the hold (timeline)
    uint32_t lk3, lrel3, rk3, rrel3;  // level-3 claim results
    uint32_t hold_on[2];           // merge leader -> merge warps: serve op j+1 (by op parity)
    unsigned long long nx_op[2], nx_off[2];
    volatile uint32_t w0_done;     // ops the control warp has finished
    volatile uint32_t w0_seen;     // op records the control warp has taken (mb_rec phases seen)
    uint32_t nb_end[8];            // node map at the hold's end
    Sv3Rec rec[4];
    // claim warp's look-ahead ring: confirmed waiting deletes by ticket % 8
    unsigned long long la_tk[8], la_op[8], la_off[8];
    // level-3 state words (slots 8-15) a claim may CAS from directly: the
    // words the server's own releases produce, and the claimed words
    uint32_t w3pred[8];
    uint32_t w3in[8];
};

struct OpShared {
    unsigned long long op;
    unsigned long long nodes;
    unsigned long long plen;
    unsigned long long seq;
    unsigned long long deleters;
    unsigned long long root_tk;  // ticket under which this CTA holds the root
    uint32_t act;
    uint32_t cw[3];     // observed state words (children / claimed node)
    uint32_t claim[3];  // 1 = claimable, 0 = skip (empty)
    uint32_t ok[3];     // CAS outcome
    uint32_t lk, rk;    // children locked?
    uint32_t lrel, rrel;  // children release states
    uint32_t lastrel;
    uint32_t owned;
    uint32_t serve;                // delete server: next ticket is a waiting delete
    unsigned long long op_next;    // its op index
    unsigned long long off_next;   // its out_pool offset
    uint32_t contw;                // served delete: continuation slot | kDelMod bit 31
    uint32_t next_w;               // delete server: pre-observed state word of the next refill
    SvPending pd;
    Sv3Shared s3;
    unsigned long long tl[16 * 24];  // profiling: per-op clocks of a three-level server (kTlSmemOps ops)
};
constexpr uint32_t kTlSmemOps = 16;

// Three-level delete server: node sizes whose 24 buffers fit in shared memory
// next to everything else, on 512-thread CTAs (16 warps: control, claim,
// 12 merge warps, 2 refill warps).  Compiled only with -DBH_SERVE3 (make
// SERVE3=1): it is an experiment, and compiled in, its
// code and its 24-buffer shared-memory footprint slow the production path
// (measured on one box: 2^26 / K=1024 insert phase 87.0 -> 85.1 ms, delete
// phase 304.7 -> 301.3 ms without it, profiles/r2/ab_final.txt).
#ifdef BH_SERVE3
constexpr bool kServe3Built = true;
#else
constexpr bool kServe3Built = false;
#endif
template <typename Key, int K, int T>
struct Serve3Cfg {
    static constexpr int kBufs = 24;
    static constexpr bool kOn =
        kServe3Built && T == 512 && (unsigned long long)kBufs * K * sizeof(Key) <= 200ull * 1024ull;
};

// Profile slots (BH_FLAG_PROFILE): SM cycles summed over ops by the leader.
enum ProfIdx {
    pfInsOps = 0,
    pfInsSort,
    pfInsRootWait,
    pfInsRootHold,
    pfInsRest,
    pfDelOps,
    pfDelRootWait,
    pfDelRootHold,
    pfDelRest,
    pfChildWait,
    pfLevels,
    pfCtaCycles,
    pfRsHead,   // delete root step: root lock -> header/root batch in smem
    pfRsChild,  //   claim + load children 2 and 3
    pfRsLast,   //   claim the last node
    pfRsLoad,   //   load the refill (+ partial)
    pfRsFill,   //   partial re-merge
    pfLvAcq,    // heapify level: claim + load children
    pfLvLoad,   //   (unused: loads overlap the claims)
    pfLvMerge,  //   both merges
    pfLvRel,    //   write-back barrier + releases
    pfServed,   // inserts served by a combiner
    pfServeHolds,  // root holds that served >= 1 waiter
    pfBuParent, // BU climb: park -> parent claimed (cycles)
    pfBuRetake, // BU climb: re-take of the parked slot (cycles)
    pfBuLevels, // BU climb levels
    pfSplitA,   // delete root split: refill half done (cycles from split start)
    pfSplitB,   // delete root split: children half done
    pfDelServed,      // deletes whose top levels a delete server ran
    pfDelServeHolds,  // root holds that served >= 1 waiting delete
    pfSvSplit,  // delete server, per op: result + refill || H0 + level-2 claims
    pfSvA,      //   refill half done (from op start)
    pfSvB,      //   H0 + claim half done (from op start)
    pfSvR1,     //   root + carried merges
    pfSvR2,     //   lo + H1 merges
    pfSvR3,     //   level-1 merges, lo2 write and release
    pfSvNext,   //   next-waiter check and continuation hand-off
    pfSvClaim,  //   level-2 claim (after H0 || lo0)
    // three-level delete server (serve3), per op, cycles
    pf3Ops,     // ops run by a three-level server
    pf3Op,      //   op barrier to op barrier
    pf3R0,      //   round 0: H0 || H1 || lo0 || lo1
    pf3WaitRf,  //   merge warps waiting for the refill batch
    pf3R1,      //   round 1: new root || carried 1
    pf3WaitC3,  //   merge warps waiting for the level-3 children
    pf3R2,      //   round 2: new hi1 || carried 2 || H2 || lo2
    pf3R3,      //   round 3: new hi2 || carried 3 (mailbox) || lo3 write
    pf3Claim,   //   claim warp: level-3 claim + load
    pf3Refill,  //   refill warps: go -> refill batch in smem
    pf3Ctl,     //   control warp: flush + result + lookups
    pf3Rec,     //   merge leader: last barrier -> record written
    pf3Wake,    //   record written -> control warp past mb_mdone
    pf3Post,    //   control warp: record -> op barrier
    pf3Start,   //   control warp at the op barrier -> round 0 starts
    pfHoldCs,   // insert root holds run by claim_and_serve: root taken -> handed on (cycles)
    pfHoldCsN,  //   their number
    pfClimbRoot,   // BU climb steps at the root: root granted -> released (cycles)
    pfClimbRootN,  //   their number
    pfCs1,      // claim_and_serve (leader, cycles): t_root -> entry
    pfCs2,      //   entry -> look-ups done
    pfCs3,      //   look-ups -> claims done
    pfCs4,      //   claims -> fence done
    kNumProf
};

// Debug builds (-DBH_DEBUG_WAIT) record, per CTA, the source line of the
// spin loop it is in and how many pauses it has made, in the profile buffer
// (words kDbgWaitBase + 4*cta ...), readable while the kernel runs.
#ifdef BH_DEBUG_WAIT
#define BH_WAIT_NOTE(line) wait_note(line)
#define BH_WAIT_NOTE2(slot, w) wait_note2(slot, w)
#define BH_OWN(slot) dbg_own(slot, __LINE__)
#else
#define BH_OWN(slot) ((void)0)
#define BH_WAIT_NOTE(line) ((void)0)
#define BH_WAIT_NOTE2(slot, w) ((void)0)
#endif
constexpr uint32_t kDbgWaitBase = 64;

// Rec: the kernel of BH_FLAG_RECORD heaps (event log); the other kernel
// carries no recording code at all.
template <typename Key, int K, int T, bool Rec>
struct HeapCta {
    static constexpr Key kMaxKey = KeyLimits<Key>::kMax;
    static constexpr int kBufs = 10;
    static constexpr uint32_t kNodeBytes = K * sizeof(Key);
    // prefetches are issued by warps other than the leader's
    static constexpr uint32_t kPfFirst = T > 64 ? 64 : 0;
    static constexpr uint32_t kRefillAhead = T > 64 ? 8 : 0;

    HeapView hv;
    RunView rv;
    Key* keys;
    uint32_t* states;
    Header* hdr;
    Key* partial;
    OpShared* sh;
    Key* bufs;
    unsigned long long cnt[kNumCounters];
    unsigned long long cur_op;
    uint32_t sv_j = 0;  // delete server: the op's index in the hold (timeline)
    bool elide;
    static constexpr bool record = Rec;
    bool prof;

    __device__ __forceinline__ HeapCta(const HeapView& h, const RunView& r, unsigned char* smem,
                                       OpShared* s)
        : hv(h), rv(r), sh(s) {
        keys = static_cast<Key*>(h.keys);
        states = h.states;
        hdr = h.hdr;
        partial = static_cast<Key*>(h.partial);
        bufs = reinterpret_cast<Key*>(smem);
#pragma unroll
        for (int i = 0; i < kNumCounters; ++i) cnt[i] = 0;
        elide = (h.flags & BH_FLAG_ELIDE_MERGES) != 0;
        prof = h.prof != nullptr;
    }

    __device__ void wait_note(int line) {
        if (!hv.prof) return;
        volatile unsigned long long* d = hv.prof + kDbgWaitBase + 4ull * blockIdx.x;
        d[0] = (unsigned long long)line | ((unsigned long long)threadIdx.x << 32);
        d[1] = d[1] + 1;
        d[2] = cur_op;
    }
    __device__ void dbg_own(unsigned long long slot, int line) {
        volatile uint32_t* o = states + slot * kStateStride;
        o[1] = (blockIdx.x + 1u) | ((uint32_t)line << 16);
        o[2] = (uint32_t)cur_op;
    }
    __device__ void wait_note2(unsigned long long slot, uint32_t w) {
        if (!hv.prof) return;
        volatile unsigned long long* d = hv.prof + kDbgWaitBase + 4ull * blockIdx.x;
        d[3] = (slot << 32) | w;
    }
    __device__ __forceinline__ Key* buf(int i) const { return bufs + i * K; }
    __device__ __forceinline__ bool leader() const { return threadIdx.x == 0; }
    __device__ __forceinline__ Key* node(unsigned long long slot) const { return keys + (slot - 1) * K; }
    __device__ __forceinline__ uint32_t* st(unsigned long long slot) const {
        return states + slot * kStateStride;
    }
    __device__ __forceinline__ void count(int idx, unsigned long long v = 1) {
        if (leader()) cnt[idx] += v;
    }
    __device__ __forceinline__ unsigned long long now() const {
        if (!prof) return 0ull;
        unsigned long long c;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");  // not moved across memory ops
        return c;
    }
    // per-op timeline of a three-level server (profiling handles): the SM
    // clock at event `ev` of the hold's op j, for ops [kTlFirst, +kTlOps)
    // Clocks go to shared memory (sh->tl) and are copied out at the hold's
    // end: a global store between two clock reads would put its own latency
    // into the next reading.
    __device__ __forceinline__ void tl(uint32_t j, uint32_t ev) {
        if (prof && j - kTlFirst < kTlSmemOps) {
            unsigned long long c;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
            sh->tl[(j - kTlFirst) * 24u + ev] = c;
        }
    }
    // profile slots go straight to global memory (a red per event, profiling
    // builds only): no per-CTA register array
    __device__ __forceinline__ void pf_add(int idx, unsigned long long v) {
        if (prof && leader()) atomicAdd(&hv.prof[idx], v);
    }
    // per-level climb profile: `what` 0 = steps, 1 = parent-claim cycles,
    // 2 = claim-to-release cycles; `parent` = the slot claimed
    __device__ __forceinline__ void pf_lv(uint32_t what, unsigned long long parent, unsigned long long v) {
        if (prof && leader())
            atomicAdd(&hv.prof[kLvBase + what * kLvLevels + (63u - (uint32_t)__clzll((long long)parent))], v);
    }
    __device__ __forceinline__ void prefetch_node(unsigned long long slot) {
        if (slot > hv.slot_count) return;
        cta_prefetch_l2<T>(node(slot), kNodeBytes, kPfFirst);
        if (threadIdx.x == kPfFirst + 32 % T) asm volatile("prefetch.global.L2 [%0];" ::"l"(st(slot)));
    }

    // ----------------------------------------------------------- recorder --
    // Recorder::op_begin/lock_acquired/lock_released/op_end
    // (proj/src/instrumentation.cpp:47-107): one global device clock.  Any
    // lane may record (children are claimed by two lanes).
    __device__ void rec_lane(uint16_t kind, unsigned long long slot) {
        if (!record) return;
        const unsigned long long ts = atomicAdd(&hdr->clock, 1ull);
        const uint32_t idx = atomicAdd(&rv.event_counts[cur_op], 1u);
        if (idx >= rv.ev_per_op) {
            atomicOr(&hdr->error_flags, (unsigned long long)kErrEventOverflow);
            return;
        }
        DevEvent& e = rv.events[cur_op * rv.ev_per_op + idx];
        e.ts = ts;
        e.op = (uint32_t)cur_op;
        e.kind = kind;
        e.pad = 0;
        e.node = slot;
    }
    __device__ void rec_for(unsigned long long op, uint16_t kind, unsigned long long slot) {
        const unsigned long long saved = cur_op;
        cur_op = op;
        rec_lane(kind, slot);
        cur_op = saved;
    }
    __device__ __forceinline__ void rec(uint16_t kind, unsigned long long slot) {
        if (record && leader()) rec_lane(kind, slot);
    }
    __device__ void rec_abort() {
        if (record && leader()) atomicExch(&rv.event_counts[cur_op], 0u);
    }

    // -------------------------------------------------------------- locks --
    // The root only ever takes AVAIL <-> INUSE (every op starts there and no
    // walk treats it as a child or refill source), so its lock is a FIFO
    // array queue lock: each waiter spins on its own 128-byte flag instead
    // of every CTA hammering one L2 word with CAS, and the hand-off costs one
    // store.  Mutual exclusion and FIFO hand-off order are the reference's
    // lock_avail(1)/unlock(1) semantics (heap.cpp:98-114).  Leader lane only.
    // Queue slot line of ticket t: word 0 = hand-off flag (t<<1 granted,
    // t<<1|1 served by a combiner), word 1 = request word (t<<1|1 when the
    // waiter is a combinable insert), words 2-3 = its op index, words 4-9 =
    // the combiner's response to an insert (rank, target slot, root
    // sequence); word 11 = request word of a servable delete (t<<1|1), whose
    // delete server writes words 0-1 at once: flag | continuation word << 32.
    __device__ __forceinline__ uint32_t* qline(unsigned long long t) const {
        return hv.root_flags + (t % kRootQueue) * kRootFlagStride;
    }
    // Returns true when a combiner ran this op's root phase instead of
    // granting the lock (combinable = a BU full-batch insert, see
    // serve_inserts).
    __device__ bool root_lock(bool record_it = true, bool combinable = false, bool del_req = false) {
        const unsigned long long t = atomicAdd(&hdr->root_tail, 1ull);
        uint32_t* f = qline(t);
        if (combinable || del_req) {
            st_cg_u64(reinterpret_cast<unsigned long long*>(f + 2), cur_op);
            // a delete server serves only ops of its own launch (its ops,
            // out_pool and status arrays), an insert combiner of a recorded
            // heap too (it logs the waiter's events): words 12-13 name the launch
            st_cg_u64(reinterpret_cast<unsigned long long*>(f + 12), (unsigned long long)rv.ticket);
            // a servable delete also names its result slot (words 4-5)
            if (del_req) st_cg_u64(reinterpret_cast<unsigned long long*>(f + 4), rv.ops[cur_op].offset);
            state_store_release(f + (del_req ? 11 : 1), ((uint32_t)t << 1) | 1u);
        }
        const uint32_t granted = (uint32_t)t << 1;
        uint32_t v;
        if (del_req) {
            // words 0-1 in one load: a delete server's hand-off puts the
            // continuation word (serve_deletes) next to the flag
            QuickBackoff b(&hdr->error_flags);
            unsigned long long vv;
            while ((((uint32_t)(vv = ld_acquire_u64(reinterpret_cast<const unsigned long long*>(f)))) & ~1u) !=
                   granted) {
                b.pause();
                BH_WAIT_NOTE(__LINE__);
            }
            v = (uint32_t)vv;
            sh->contw = (uint32_t)(vv >> 32);
        } else {
            // (no sleeps either: each waiter polls its own line, and the
            // root hand-off is on the insert phase's chain -- 256 ns sleeps
            // cost the 2^26 / K=1024 insert phase ~1.3 ms,
            // profiles/r2/ab_final.txt)
            QuickBackoff b(&hdr->error_flags);
            while (((v = state_load(f)) & ~1u) != granted) { b.pause(); BH_WAIT_NOTE(__LINE__); }
        }
        sh->root_tk = t;
        if (v & 1u) return true;
        if (record_it) rec_lane(kEvAcq, 1);
        return false;
    }
    __device__ void root_unlock(bool record_it = true) {
        if (record_it) rec_lane(kEvRel, 1);
        const unsigned long long nt = sh->root_tk + 1;
        state_store_release(qline(nt), (uint32_t)nt << 1);
    }

    // Insert combining (flat combining inside the queue lock).  A BU full-
    // batch insert holding the root, with the partial buffer empty, also runs
    // the root phase of the queued waiters behind it that are BU full-batch
    // inserts: each gets the next rank and its bit-reversed target slot,
    // claimed INUSE under the root lock exactly as its own root phase would
    // (heap.cpp:126-188, 295-308), in queue order -- so each op still
    // linearizes at its rank assignment, one after the other, inside this
    // root hold.  The waiter is woken with its response instead of the lock
    // and goes straight to writing its target and climbing.  Warp 0, root
    // held, own target claimed.  Returns the number of ops served.
    __device__ uint32_t serve_inserts(unsigned long long nodes_after, unsigned long long seq_next) {
        const uint32_t lane = threadIdx.x & 31u;
        unsigned long long tail = 0;
        if (lane == 0) tail = ld_cg_u64(&hdr->root_tail);
        tail = __shfl_sync(0xFFFFFFFFu, tail, 0);
        const unsigned long long mine = sh->root_tk;
        const unsigned long long t = mine + 1 + lane;
        uint32_t* f = qline(t);
        bool ok = t < tail && nodes_after + 1 + lane <= hv.max_nodes;
        unsigned long long op = 0;
        if (ok) {
            ok = state_load(f + 1) == (((uint32_t)t << 1) | 1u);
            if (ok && record)
                ok = ld_cg_u64(reinterpret_cast<const unsigned long long*>(f + 12)) == (unsigned long long)rv.ticket;
            if (ok) op = ld_cg_u64(reinterpret_cast<const unsigned long long*>(f + 2));
        }
        const uint32_t bad = __ballot_sync(0xFFFFFFFFu, !ok);
        const uint32_t g = bad ? (uint32_t)__ffs(bad) - 1u : 32u;
        unsigned long long target = 0;
        if (lane < g) {
            const unsigned long long rank = nodes_after + 1 + lane;
            target = slot_for_rank(rank);
            lane_claim(target, (1u << kAvail) | (1u << kDelMod));
            st_cg_u64(reinterpret_cast<unsigned long long*>(f + 4), rank);
            st_cg_u64(reinterpret_cast<unsigned long long*>(f + 6), target);
            st_cg_u64(reinterpret_cast<unsigned long long*>(f + 8), seq_next + lane);
        }
        __syncwarp();
        if (record) {  // each served op's root span, one after the other
            for (uint32_t i = 0; i < g; ++i) {
                const unsigned long long oi = __shfl_sync(0xFFFFFFFFu, op, i);
                const unsigned long long ti = __shfl_sync(0xFFFFFFFFu, target, i);
                if (lane == 0) {
                    rec_for(oi, kEvAcq, 1);
                    rec_for(oi, kEvAcq, ti);
                    rec_for(oi, kEvRel, 1);
                }
                __syncwarp();
            }
        }
        if (lane < g) state_store_release(f, ((uint32_t)t << 1) | 1u);
        return g;
    }

    // insert_bu's own target claim and insert combining in one pass
    // (unrecorded heaps; recorded ones log each step through the two calls
    // above).  Warp 0, root held, partial buffer empty: lane 0 claims this
    // op's target (rank), lanes 1..31 the targets of the queued BU full-batch
    // inserts behind it (ranks rank+1.., in ticket order), with the look-ups
    // (queue tail, request words, target state words) in one round of loads
    // and the claims in one round of CASes; then the leader publishes the
    // responses, the header and the hand-offs behind one fence and lets the
    // root go.  Same ranks, targets, states, sequence numbers and FIFO
    // hand-off as the claim + serve_inserts + root_unlock it replaces
    // (heap.cpp:126-188, 295-308).  Sets cur_word on every lane.
    __device__ void claim_and_serve(unsigned long long target, unsigned long long rank, unsigned long long seq,
                                    uint32_t& cur_word, unsigned long long t_root) {
        const uint32_t lane = threadIdx.x & 31u;
        const unsigned long long tcs0 = now();
        pf_add(pfCs1, tcs0 - t_root);
        const unsigned long long mine = sh->root_tk;
        const unsigned long long t = mine + lane;  // lane 0: this op's own ticket
        uint32_t* f = qline(t);
        const unsigned long long rk = rank + lane;
        const bool fits = rk <= hv.max_nodes;  // lane 0: checked by do_insert
        const unsigned long long tg = lane ? (fits ? slot_for_rank(rk) : 0ull) : target;
        // round 1
        // (the target words are only the CASes' expected values: relaxed,
        // issued ahead of the one acquire, so all three travel together)
        const uint32_t tw = fits ? state_poll(st(tg)) : 0u;
        unsigned long long tail = 0;
        if (lane == 0) tail = ld_cg_u64(&hdr->root_tail);
        const uint32_t req = (lane && fits) ? state_load(f + 1) : 0u;
        tail = __shfl_sync(0xFFFFFFFFu, tail, 0);
        const bool ok = lane == 0 || (fits && t < tail && req == (((uint32_t)t << 1) | 1u));
        const uint32_t bad = __ballot_sync(0xFFFFFFFFu, !ok);
        const uint32_t n = bad ? (uint32_t)__ffs(bad) - 1u : 32u;  // lanes [0, n) claim
        const unsigned long long tcs1 = now();
        pf_add(pfCs2, tcs1 - tcs0);
        // round 2: the claims
        uint32_t got = 0;
        if (lane < n) {
            const uint32_t st0 = sget(tw);
            // relaxed: the leader's fence below orders the claims before
            // every hand-off and before any write to the targets
            if ((st0 == kAvail || st0 == kDelMod) && state_cas_relaxed(st(tg), tw, swith(tw, kInUse))) {
                BH_OWN(tg);
                got = swith(tw, kInUse);
            } else {
                lane_claim(tg, (1u << kAvail) | (1u << kDelMod), &got);
            }
        }
        cur_word = __shfl_sync(0xFFFFFFFFu, got, 0);
        const unsigned long long tcs2 = now();
        pf_add(pfCs3, tcs2 - tcs1);
        const uint32_t g = n - 1u;  // ops served
        if (lane && lane < n) {
            st_cg_u64(reinterpret_cast<unsigned long long*>(f + 4), rk);
            st_cg_u64(reinterpret_cast<unsigned long long*>(f + 6), tg);
            st_cg_u64(reinterpret_cast<unsigned long long*>(f + 8), seq + lane);
        }
        __syncwarp();
        if (lane == 0) {
            if (g) {
                st_cg_u64(&hdr->node_count, rank + g);
                st_cg_u64(&hdr->root_seq, seq + 1 + g);
                atomicAdd(gate_mine(true), (unsigned long long)g);
                count(cCombined, g);
                pf_add(pfServed, g);
                pf_add(pfServeHolds, 1);
            }
            __threadfence();  // claims, responses, header and gate count before any hand-off
            pf_add(pfCs4, now() - tcs2);
            for (uint32_t i = 1; i <= g; ++i)
                state_store_relaxed(qline(mine + i), ((uint32_t)(mine + i) << 1) | 1u);
            const unsigned long long nt = mine + g + 1;  // root_unlock
            sh->root_tk = mine + g;
            state_store_relaxed(qline(nt), (uint32_t)nt << 1);
            pf_add(pfHoldCs, now() - t_root);
            pf_add(pfHoldCsN, 1);
        }
        __syncwarp();
    }

    // Non-root claim: wait for one of `accept` (bitmask of states), CAS it to
    // INUSE.  Returns the state it was claimed from.  Calling lane only.
    __device__ uint32_t lane_claim(unsigned long long slot, uint32_t accept, uint32_t* claimed_word = nullptr) {
        uint32_t* p = st(slot);
        Backoff b(&hdr->error_flags);
        for (;;) {
            const uint32_t w = state_load(p);
            if (((accept >> sget(w)) & 1u) && state_cas(p, w, swith(w, kInUse))) {
                BH_OWN(slot);
                if (claimed_word) *claimed_word = swith(w, kInUse);
                return sget(w);
            }
            { b.pause(); BH_WAIT_NOTE(__LINE__); }
        }
    }
    // unlock (heap.cpp:111-114) of a node this lane's CTA holds INUSE.  The
    // CTA has passed a barrier after its last write to the node.
    __device__ __forceinline__ void lane_unlock(unsigned long long slot, uint32_t release_as = kAvail) {
        if (slot == 1) {
            root_unlock();
            return;
        }
        rec_lane(kEvRel, slot);
#ifdef BH_DEBUG_WAIT
        { volatile uint32_t* o = states + slot * kStateStride; o[1] = 0xDEAD0000u | (uint32_t)(blockIdx.x & 0xFFFF); }
#endif
        state_release(st(slot), kInUse, release_as);
    }

    // ---------------------------------------------------- BU phase gate --
    // Deviation from the reference (SURVEY.md section 4 lists its other
    // bugs): in BU heaps a bottom-up climb and a delete's heapify never run
    // at the same time.  The reference lets deleters take over slots parked
    // mid-climb (INSHOLD -> DELMOD, heap.cpp:508-516,567-573); a random-
    // interleaving model of that protocol (tools/sim_bu.py) breaks property 1
    // in ~0.5% of schedules (the owner loses its park to another climber's
    // DELMOD consumption, or skips re-checking a slot a deleter only took as
    // its lo child), and the GPU reproduced it.  It also covers partial-
    // buffer keys a full batch absorbs: visible before the climb, they would
    // be hidden from concurrent deletes during it (non-linearizable
    // histories, found by the exhaustive checker).  Insert-only and
    // delete-only concurrency are each safe, so an op of one kind that finds
    // the other kind in flight lets the root go and queues again.
    __device__ __forceinline__ unsigned long long* gate_mine(bool climb) {
        return climb ? &hdr->climbers : &hdr->deleters;
    }
    __device__ __forceinline__ unsigned long long* gate_other(bool climb) {
        return climb ? &hdr->deleters : &hdr->climbers;
    }
    // Phase token (root-lock guarded).  Ops of the open phase enter until an
    // op of the other kind arrives and closes it; that op (and its kind)
    // wait outside the root queue until the running kind has drained, then
    // the first of them flips the phase and its whole batch enters.  Leader
    // lane, root held.  Returns true when the op may start (counted).
    __device__ bool gate_try(bool climb) {
        return gate_try(climb, ld_cg_u64(&hdr->gate_phase), ld_cg_u64(&hdr->gate_closing),
                        ld_cg_u64(gate_other(climb)));
    }
    // With the gate words already loaded under the root lock (phase and
    // closing only change under it; the other kind's count only falls
    // outside it, so an early read errs on the waiting side).
    __device__ bool gate_try(bool climb, unsigned long long ph, unsigned long long closing,
                             unsigned long long other) {
        if (hv.flags & kDbgNoGate) {  // measurement only: what the gate costs
            atomicAdd(gate_mine(climb), 1ull);
            return true;
        }
        const unsigned long long me = climb ? 0ull : 1ull;
        if (ph == me && !closing) {
            atomicAdd(gate_mine(climb), 1ull);  // ordered before the root release
            return true;
        }
        if (ph != me && other == 0) {
            st_cg_u64(&hdr->gate_phase, me);
            st_cg_u64(&hdr->gate_closing, 0ull);
            atomicAdd(gate_mine(climb), 1ull);
            return true;
        }
        if (ph != me) st_cg_u64(&hdr->gate_closing, 1ull);
        return false;
    }
    // Wait (root not held, not queued) until a retry can succeed or can
    // close the running phase.
    __device__ void gate_wait(bool climb) {
        const unsigned long long me = climb ? 0ull : 1ull;
        Backoff b(&hdr->error_flags);
        for (;;) {
            const unsigned long long ph = __ldcg(&hdr->gate_phase);
            const unsigned long long closing = __ldcg(&hdr->gate_closing);
            const unsigned long long other = __ldcg(gate_other(climb));
            if (ph == me ? !closing : (other == 0 || !closing)) return;
            { b.pause(); BH_WAIT_NOTE(__LINE__); }
        }
    }
    __device__ void gate_leave(bool climb) {
        __threadfence();
        atomicAdd(gate_mine(climb), ~0ull);  // -1, after every write of the op
    }

    __device__ void status(unsigned long long opi, uint32_t code, uint32_t len, unsigned long long seq) {
        if (!leader()) return;
        if (rv.out_status) rv.out_status[opi] = code;
        if (rv.out_lens) rv.out_lens[opi] = len;
        if (rv.out_seq) rv.out_seq[opi] = seq;
    }

    __device__ void note_partial(unsigned long long len) {
        if (leader() && len > cnt[cMaxPartial]) cnt[cMaxPartial] = len;
    }

    // =============================================================== run ==
    __device__ void run() {
        const unsigned long long t_start = now();
        for (;;) {
            if (leader()) sh->op = atomicAdd(rv.ticket, 1ull);
            __syncthreads();
            const unsigned long long opi = sh->op;
            __syncthreads();
            if (opi >= rv.n_ops) break;
            cur_op = opi;
            const bh_op o = rv.ops[opi];
            if (o.kind == BH_OP_INSERT)
                do_insert(opi, o);
            else
                do_delete(opi, o);
            __syncthreads();
        }
        pf_add(pfCtaCycles, now() - t_start);
        if (leader()) {
#pragma unroll
            for (int i = 0; i < kNumCounters; ++i) {
                if (i == cMaxPartial) {
                    if (cnt[i]) atomicMax(&hv.counters[i], cnt[i]);
                } else if (cnt[i]) {
                    atomicAdd(&hv.counters[i], cnt[i]);
                }
            }

        }
    }

    // ============================================================ insert ==
    __device__ void do_insert(unsigned long long opi, const bh_op& o) {
        const uint32_t n = o.len;
        if (n == 0 || n > (uint32_t)K) {  // sort_batch capacity errors (batch.cpp:8-12)
            status(opi, BH_E_CAPACITY, 0, ~0ull);
            return;
        }
        const unsigned long long t0 = now();
        Key* sorted = buf(0);
        const Key* src = static_cast<const Key*>(rv.key_pool) + o.offset;
        bool bad;
        if constexpr (K >= T) {
            bad = cta_sort_batch<Key, K, T>(src, n, sorted, buf(1));  // buf(1) is free until the root phase
        } else {
            int b = 0;
            for (uint32_t i = threadIdx.x; i < (uint32_t)K; i += T) {
                Key v = kMaxKey;
                if (i < n) {
                    v = src[i];
                    b |= v >= kMaxKey;
                }
                sorted[i] = v;
            }
            bad = __syncthreads_or(b) != 0;
            if (!bad) cta_bitonic_sort<Key, K, T>(sorted);
        }
        if (bad) {  // batch.cpp:13-15, before any mutation
            status(opi, BH_E_INVALID_KEY, 0, ~0ull);
            return;
        }
        rec(kEvInv, 0);
        const unsigned long long t1 = now();

        // ---- root phase (heap.cpp:126-167) ----
        if (leader()) {
            uint32_t gated = 0;
            const bool combinable =
                hv.variant == BH_BU && n == (uint32_t)K && (hv.flags & kDbgNoCombine) == 0;
            bool served = false;
            for (;;) {
                served = root_lock(false, combinable);
                if (served) break;
                // the header and (BU) the gate words in one round of loads
                const unsigned long long nd = ld_cg_u64(&hdr->node_count);
                const unsigned long long pl = ld_cg_u64(&hdr->partial_len);
                const unsigned long long sq = ld_cg_u64(&hdr->root_seq);
                unsigned long long gph = 0, gcl = 0, got = 0;
                if (hv.variant == BH_BU) {
                    gph = ld_cg_u64(&hdr->gate_phase);
                    gcl = ld_cg_u64(&hdr->gate_closing);
                    got = ld_cg_u64(gate_other(true));
                }
                sh->nodes = nd;
                sh->plen = pl;
                sh->seq = sq;
                // a BU full batch with rank >= 2 climbs: phase gate
                const bool climbs = hv.variant == BH_BU && n + (uint32_t)pl >= (uint32_t)K && nd >= 1 &&
                                    nd < hv.max_nodes;
                if (!climbs) break;
                if (gate_try(true, gph, gcl, got)) {
                    gated = 1;
                    break;
                }
                root_unlock(false);
                gate_wait(true);
            }
            if (served) {
                // a combiner ran the root phase: rank, claimed target, sequence
                const unsigned long long* f =
                    reinterpret_cast<const unsigned long long*>(qline(sh->root_tk));
                sh->nodes = ld_cg_u64(f + 2) - 1;  // words 4-5: rank
                sh->plen = 0;
                sh->seq = ld_cg_u64(f + 4);         // words 8-9
                sh->owned = 1;                      // counted in the climbers gate
                sh->act = 1;
            } else {
                rec(kEvAcq, 1);
                sh->owned = gated;
                sh->act = 0;
            }
        }
        const unsigned long long t2 = now();
        __syncthreads();
        const unsigned long long nodes = sh->nodes;
        const uint32_t plen = (uint32_t)sh->plen;
        const unsigned long long seq = sh->seq;
        const bool gated = sh->owned != 0;
        const bool served = sh->act != 0;
        const bool full = n + plen >= (uint32_t)K;
        if (full && nodes == hv.max_nodes) {  // heap.cpp:129-135
            if (leader()) lane_unlock(1);
            rec_abort();
            status(opi, BH_E_CAPACITY, 0, ~0ull);
            return;
        }
        if (leader() && !served) st_cg_u64(&hdr->root_seq, seq + 1);
        count(cInserts);
        pf_add(pfInsOps, 1);
        pf_add(pfInsSort, t1 - t0);
        pf_add(pfInsRootWait, t2 - t1);

        const uint32_t total = n + plen;
        Key* comb = sorted;  // the combined run; 2K wide when merged (buf 2..3)
        if (plen) {
            Key* part = buf(1);
            comb = buf(2);
            cta_load<Key, T>(part, partial, plen);
            __syncthreads();
            cta_merge<Key, T>(sorted, n, part, plen, comb, 2 * K, comb);
            __syncthreads();
        }

        if (!full) {
            if (nodes >= 1) {
                Key* root = buf(4);
                cta_load<Key, T>(root, node(1), K);
                __syncthreads();
                if (elide && comb[0] >= root[K - 1]) {
                    count(cElided);
                    cta_store<Key, T>(partial, comb, total);
                } else {
                    // merge_and_sort(root, combined): hi -> root, lo -> partial
                    cta_merge<Key, T>(root, K, comb, total, node(1), K, partial);
                    count(cMerges);
                }
            } else {
                cta_store<Key, T>(partial, comb, total);
            }
            note_partial(total);
            __syncthreads();
            if (leader()) {
                st_cg_u64(&hdr->partial_len, total);
                lane_unlock(1);
            }
            pf_add(pfInsRootHold, now() - t2);
            status(opi, BH_OK, 0, seq);
            rec(kEvRes, 0);
            return;
        }

        if (total > (uint32_t)K) cta_store<Key, T>(partial, comb + K, total - K);
        note_partial(total - K);
        const unsigned long long rank = nodes + 1;
        if (leader() && !served) {
            if (plen || total != (uint32_t)K) st_cg_u64(&hdr->partial_len, total - K);
            st_cg_u64(&hdr->node_count, rank);
        }
        if (rank == 1) {
            cta_store<Key, T>(node(1), comb, K);
            count(cVisits);
            __syncthreads();
            if (leader()) lane_unlock(1);
            pf_add(pfInsRootHold, now() - t2);
            status(opi, BH_OK, 0, seq);
            rec(kEvRes, 0);
            return;
        }
        const unsigned long long target = slot_for_rank(rank);
        if (hv.variant == BH_TD) {
            insert_td(target, comb, t2);
        } else {
            const bool can_serve = plen == 0 && n == (uint32_t)K && (hv.flags & kDbgNoCombine) == 0;
            insert_bu(target, comb, t2, served, can_serve, rank, seq);
            if (gated && leader()) gate_leave(true);
        }
        status(opi, BH_OK, 0, seq);
        rec(kEvRes, 0);
    }

    // merge_step_down (heap.cpp:190-205): node `slot` keeps the k smallest of
    // node U batch; the batch keeps the rest.  `nd` must already hold the
    // node's keys (barrier passed).  Rotates bat/nd/tmp.  Ends with a barrier.
    __device__ void merge_step_down(Key*& bat, Key*& nd, Key*& tmp, unsigned long long slot) {
        if (slot != 1 && nd[0] == kMaxKey && leader())
            atomicOr(&hdr->error_flags, (unsigned long long)kErrInteriorEmpty);
        if (elide && !needs_merge_full<Key, K>(nd, bat)) {
            count(cElided);
            if (!(nd[K - 1] <= bat[0])) {
                cta_store<Key, T>(node(slot), bat, K);  // swap
                Key* t = bat;
                bat = nd;
                nd = t;
            }
        } else {
            cta_merge_full_bt<Key, K, T>(nd, bat, node(slot), tmp);
            count(cMerges);
            Key* t = bat;
            bat = tmp;
            tmp = t;
        }
        __syncthreads();
    }

    // insert_td (heap.cpp:218-293).  Root held on entry.
    __device__ void insert_td(unsigned long long target, Key* bat, unsigned long long t_root) {
        Key* nd = buf(4);
        Key* tmp = buf(5);
        // claim the target under the root lock: AVAIL -> TARGET (leader)
        auto claim_target = [&]() {
            uint32_t* p = st(target);
            Backoff b(&hdr->error_flags);
            for (;;) {
                // relaxed: nothing of the target is read, and its write comes
                // after the root's release (a fence) further down
                const uint32_t w = state_poll(p);
                const uint32_t s = sget(w);
                // (DELMOD: BU heaps only; never seen in TD heaps)
                if ((s == kAvail || s == kDelMod) && state_cas_relaxed(p, w, swith(w, kTarget))) break;
                { b.pause(); BH_WAIT_NOTE(__LINE__); }
            }
        };
        const int depth = (int)level_of(target);
        // Below level 1 the claim rides with the first child's: its word
        // loads beside the child's poll and its CAS beside the child's, after
        // the root's merge, still under the root (the reference claims it
        // before that merge, heap.cpp:220-230); two round trips off the hold.
        uint32_t tpend = depth >= 2 ? 1u : 0u, tw = 0;
        if (leader() && !tpend) claim_target();
        cta_load<Key, T>(nd, node(1), K);  // root keys, in the claim's round trip
        __syncthreads();
        merge_step_down(bat, nd, tmp, 1);
        count(cVisits);
        unsigned long long cur = 1;
        enum { kShip = 1, kWrite = 2, kSkip = 3, kMerge = 4 };
        for (int lvl = depth - 1; lvl >= 0;) {
            const unsigned long long next = target >> lvl;
            if (leader()) {
                uint32_t act = 0;
                if (tpend) tw = state_poll(st(target));
                if (cur != 1 && sget(state_load(st(target))) == kMarked) {
                    act = kShip;
                } else if (next == target) {
                    Backoff b(&hdr->error_flags);
                    for (;;) {
                        const uint32_t w = state_load(st(target));
                        if (sget(w) == kTarget) {
                            if (state_cas(st(target), w, swith(w, kInUse))) {
                                act = kWrite;
                                break;
                            }
                        } else if (sget(w) == kMarked) {
                            act = kShip;
                            break;
                        } else {
                            { b.pause(); BH_WAIT_NOTE(__LINE__); }
                        }
                    }
                } else {
                    Backoff b(&hdr->error_flags);
                    for (;;) {
                        const uint32_t w = state_load(st(next));
                        const uint32_t s = sget(w);
                        if (s == kAvail) {
                            act = kMerge;  // claimed below, overlapped with the load
                            sh->cw[0] = w;
                            break;
                        } else if (s == kTarget || s == kMarked) {
                            act = kSkip;  // frozen empty while we hold its ancestor
                            break;
                        } else {
                            { b.pause(); BH_WAIT_NOTE(__LINE__); }
                        }
                    }
                }
                if (tpend && act != kMerge) {
                    claim_target();
                    tpend = 0;
                }
                sh->act = act;
            }
            __syncthreads();
            const uint32_t act = sh->act;
            if (act == kShip) {  // ship_to_root (heap.cpp:207-216)
                cta_store<Key, T>(node(1), bat, K);
                count(cCoop);
                __syncthreads();
                if (leader()) {
                    state_release(st(target), kMarked, kAvail);
                    lane_unlock(cur);
                }
                if (cur == 1) pf_add(pfInsRootHold, now() - t_root);
                return;
            }
            if (act == kWrite) {
                if (leader()) {
                    rec(kEvAcq, target);
                    lane_unlock(cur);
                }
                if (cur == 1) pf_add(pfInsRootHold, now() - t_root);
                cta_store<Key, T>(node(target), bat, K);
                count(cVisits);
                __syncthreads();
                if (leader()) lane_unlock(target);
                return;
            }
            if (act == kSkip) {
                --lvl;
                continue;
            }
            // kMerge: load the node while the leader's CAS claims it
            uint32_t ok = 0, okt = 1;
            if (leader()) {
                const uint32_t w = sh->cw[0];
                ok = state_cas_relaxed(st(next), w, swith(w, kInUse));
                if (tpend) {
                    const uint32_t s = sget(tw);
                    okt = (s == kAvail || s == kDelMod) && state_cas_relaxed(st(target), tw, swith(tw, kTarget));
                }
            }
            cta_load<Key, T>(nd, node(next), K);
            if (leader()) {
                sh->ok[0] = ok;
                if (tpend) {
                    if (!okt) claim_target();
                    tpend = 0;
                }
            }
            __syncthreads();
            if (!sh->ok[0]) continue;  // lost the race: decide again
            // hand over hand: the parent goes as soon as the child is held
            // (its batch is final, written by the previous step); the
            // reference unlocks it after merging at the child
            // (heap.cpp:281-288), the same lock order, and a waiter on
            // the parent still meets the child held until this merge is in
            if (leader()) {
                rec(kEvAcq, next);
                lane_unlock(cur);
            }
            if (cur == 1) pf_add(pfInsRootHold, now() - t_root);
            merge_step_down(bat, nd, tmp, next);
            count(cVisits);
            cur = next;
            --lvl;
        }
    }

    // abandon_park (heap.cpp:393-407).  Calling lane only.
    __device__ void lane_abandon_park(unsigned long long slot) {
        Backoff b(&hdr->error_flags);
        uint32_t* p = st(slot);
        for (;;) {
            const uint32_t w = state_load(p);
            const uint32_t s = sget(w);
            if (s == kDelMod) {
                if (state_cas(p, w, swith(w, kAvail) + 8u)) return;
            } else if (s != kInUse) {
                return;  // AVAIL, or a later insert owns the slot now
            } else {
                { b.pause(); BH_WAIT_NOTE(__LINE__); }
            }
        }
    }

    // insert_bu (heap.cpp:295-373).  Root held on entry.
    // `served`: a combiner already claimed the target (serve_inserts);
    // `can_serve`: this op may combine the waiters behind it.
    __device__ void insert_bu(unsigned long long target, Key* bat, unsigned long long t_root, bool served,
                              bool can_serve, unsigned long long rank, unsigned long long seq) {
        Key* par = bat == buf(4) ? buf(1) : buf(4);
        Key* cu = buf(5);
        uint32_t cur_word = 0;  // leader: exact state word of the held `cur` (0 = unknown)
        if (!served && can_serve && !record) {
            if (threadIdx.x < 32) claim_and_serve(target, rank, seq, cur_word, t_root);
        } else if (!served) {
            if (leader()) {
                lane_claim(target, (1u << kAvail) | (1u << kDelMod), &cur_word);
                rec(kEvAcq, target);
            }
            if (can_serve && threadIdx.x < 32) {
                __syncwarp();
                if (leader()) rec_lane(kEvRel, 1);  // this op's own root span ends here
                const uint32_t g = serve_inserts(rank, seq + 1);
                if (leader()) {
                    if (g) {
                        st_cg_u64(&hdr->node_count, rank + g);
                        st_cg_u64(&hdr->root_seq, seq + 1 + g);
                        atomicAdd(gate_mine(true), (unsigned long long)g);
                        sh->root_tk += g;
                        count(cCombined, g);
                        pf_add(pfServed, g);
                        pf_add(pfServeHolds, 1);
                    }
                    // The target is ours (INUSE): let the root go before writing it.
                    root_unlock(false);
                }
            } else if (leader()) {
                // The target is ours (INUSE): let the root go before writing it.
                root_unlock();
            }
        }
        pf_add(pfInsRootHold, now() - t_root);
        const unsigned long long t3 = now();
        __syncthreads();  // nobody writes the target before the claim above
        cta_store<Key, T>(node(target), bat, K);
        count(cVisits);
        __syncthreads();

        unsigned long long cur = target;  // held
        if (!(hv.flags & kDbgParkClimb)) {
            climb_gated(cur, bat, par, cur_word, t3);
            return;
        }
        while (cur != 1) {
            const unsigned long long parent = cur >> 1;
            const unsigned long long tc0 = now();
            pf_add(pfBuLevels, 1);
            // ---- park, then claim the parent with its keys in flight ----
            if (leader()) lane_unlock(cur, kInsHold);
            for (;;) {
                if (leader()) {
                    if (parent == 1) {
                        root_lock();
                        sh->ok[0] = 2;  // held, nothing to validate
                    } else {
                        uint32_t* pp = st(parent);
                        Backoff b(&hdr->error_flags);
                        uint32_t w;
                        for (;;) {
                            w = state_load(pp);
                            if (sget(w) == kAvail || sget(w) == kDelMod) break;
                            { b.pause(); BH_WAIT_NOTE(__LINE__); }
                        }
                        sh->cw[0] = w;
                        sh->ok[0] = 0;
                    }
                }
                __syncthreads();
                uint32_t ok = 1;
                if (leader() && sh->ok[0] == 0) {
                    const uint32_t w = sh->cw[0];
                    ok = state_cas_relaxed(st(parent), w, swith(w, kInUse));
                }
                cta_load<Key, T>(par, node(parent), K);
                if (leader() && sh->ok[0] == 0) sh->ok[0] = ok;
                __syncthreads();
                if (sh->ok[0]) break;
            }
            if (parent != 1 && leader()) rec(kEvAcq, parent);
            const unsigned long long tc1 = now();
            pf_add(pfBuParent, tc1 - tc0);
            pf_lv(0, parent, 1);
            pf_lv(1, parent, tc1 - tc0);
            if (par[0] == kMaxKey) {
                // parent was deleted: the subtree with our parked slot is gone
                if (leader()) {
                    lane_unlock(parent);
                    lane_abandon_park(cur);
                }
                pf_add(pfInsRest, now() - t3);
                return;
            }
            // ---- re-take the parked slot; its keys load with the CAS ----
            for (;;) {
                if (leader()) {
                    uint32_t* pc = st(cur);
                    Backoff b(&hdr->error_flags);
                    uint32_t owned = 0;
                    for (;;) {
                        const uint32_t w = state_load(pc);
                        const uint32_t s = sget(w);
                        if (s == kInsHold) {
                            sh->cw[1] = w;
                            owned = 1;  // provisional: validated by the CAS
                            break;
                        } else if (s == kDelMod) {
                            if (state_cas(pc, w, swith(w, kAvail) + 8u)) break;
                        } else if (s != kInUse) {
                            break;  // AVAIL (or re-claimed): consumed
                        } else {
                            { b.pause(); BH_WAIT_NOTE(__LINE__); }  // INUSE: a deleter is working on it
                        }
                    }
                    sh->owned = owned;
                }
                __syncthreads();
                if (!sh->owned) break;
                uint32_t ok = 0;
                if (leader()) {
                    const uint32_t w = sh->cw[1];
                    ok = state_cas_relaxed(st(cur), w, swith(w, kInUse));
                }
                cta_load<Key, T>(cu, node(cur), K);
                if (leader()) sh->ok[1] = ok;
                __syncthreads();
                if (sh->ok[1]) break;
            }
            pf_add(pfBuRetake, now() - tc1);
            if (sh->owned) {
                if (leader()) rec(kEvAcq, cur);
                if (cu[0] >= par[K - 1]) {
                    count(cEarlyStops);
                    if (leader()) {
                        lane_unlock(cur);
                        lane_unlock(parent);
                    }
                    pf_add(pfInsRest, now() - t3);
                    return;
                }
                // merge_step_up (heap.cpp:375-391): parent keeps the k smallest
                if (elide && !needs_merge_full<Key, K>(cu, par)) {
                    count(cElided);
                    cta_store<Key, T>(node(parent), cu, K);
                    cta_store<Key, T>(node(cur), par, K);
                } else {
                    cta_merge_full_bt<Key, K, T>(cu, par, node(parent), node(cur));
                    count(cMerges);
                }
                count(cVisits);
                __syncthreads();
                if (leader()) lane_unlock(cur);
            }
            cur = parent;
        }
        if (leader()) lane_unlock(1);
        pf_add(pfInsRest, now() - t3);
    }

    // The bottom-up climb (heap.cpp:310-391) under the BU phase gate.  Same
    // states, transitions and lock order as the reference -- park the slot
    // (INUSE -> INSHOLD), claim the parent, re-take the slot (INSHOLD ->
    // INUSE), early stop or merge_step_up, release the slot -- but the gate
    // guarantees no delete heapify runs during a climb, so nobody else ever
    // touches a parked slot.  Hence:
    //   * the park carries no data and is a relaxed red (no release fence);
    //   * the climber keeps the batch of the node it holds in shared memory
    //     and re-takes the parked slot with a CAS on the exact word it parked,
    //     without reloading the keys and without waiting for the CAS before
    //     merging (its result is checked before any write to the slot);
    //   * the node it carries up is written once, when it is released;
    //   * the release fence of each finished slot is paid by another warp.
    // `cu` holds the held node's batch on entry (the target's, already in
    // HBM); cur_word is the leader's view of cur's state word (0 if unknown).
    __device__ void climb_gated(unsigned long long cur, Key* cu, Key* par, uint32_t cur_word,
                                unsigned long long t3) {
        constexpr uint32_t kRelLane = T >= 64 ? 32 : 0;
        auto bidx = [this](const Key* b) { return (int)((b - bufs) / K); };
        int ci = bidx(cu), pi = bidx(par);
        const int si = 7;  // staging for the slot's new batch
        int ni = __ffs(~((1u << ci) | (1u << pi) | (1u << si))) - 1;
        bool cur_written = true;  // the target's batch is already in HBM
        unsigned long long t_rg = 0;  // leader: root granted (profile)
        while (cur != 1) {
            const unsigned long long parent = cur >> 1;
            const unsigned long long tc0 = now();
            pf_add(pfBuLevels, 1);
            uint32_t parked = 0;
            if (leader()) {
                rec_lane(kEvRel, cur);
                if (cur_word) {
                    state_release_relaxed(st(cur), kInUse, kInsHold);
                    parked = swith(cur_word, kInsHold) + 8u;  // the word the park leaves
                } else {
                    state_release(st(cur), kInUse, kInsHold);
                }
            }
            // ---- claim the parent with its keys in flight ----
            for (;;) {
                if (leader()) {
                    if (parent == 1) {
                        root_lock();
                        t_rg = now();
                        sh->ok[0] = 2;
                    } else {
                        uint32_t* pp = st(parent);
                        Backoff b(&hdr->error_flags);
                        uint32_t w;
                        for (;;) {
                            w = state_load(pp);
                            if (sget(w) == kAvail || sget(w) == kDelMod) break;
                            { b.pause(); BH_WAIT_NOTE(__LINE__); }
                        }
                        sh->cw[0] = w;
                        sh->ok[0] = 0;
                    }
                }
                __syncthreads();
                uint32_t ok = 1;
                if (leader() && sh->ok[0] == 0) {
                    const uint32_t w = sh->cw[0];
                    ok = state_cas_relaxed(st(parent), w, swith(w, kInUse));
                }
                cta_load<Key, T>(buf(pi), node(parent), K);
                if (leader() && sh->ok[0] == 0) sh->ok[0] = ok;
                __syncthreads();
                if (sh->ok[0]) break;
                __syncthreads();  // (a retry: everyone has read sh->ok before the leader rewrites it)
            }
            uint32_t parent_word = 0;
            if (leader() && parent != 1) {
                rec(kEvAcq, parent);
                parent_word = swith(sh->cw[0], kInUse);
            }
            const unsigned long long tc1 = now();
            pf_add(pfBuParent, tc1 - tc0);
            pf_lv(0, parent, 1);
            pf_lv(1, parent, tc1 - tc0);
            Key* P = buf(pi);
            Key* C = buf(ci);
            // ---- re-take the parked slot (CAS in flight while we merge) ----
            uint32_t retake_ok = 1;
            if (leader()) {
                if (parked) {
                    retake_ok = state_cas_relaxed(st(cur), parked, swith(parked, kInUse));
                    cur_word = swith(parked, kInUse);
                } else {
                    // word unknown (a combiner claimed the target): poll it
                    uint32_t* pc = st(cur);
                    uint32_t w;
                    Backoff b(&hdr->error_flags);
                    while (sget(w = state_load(pc)) != kInsHold) { b.pause(); BH_WAIT_NOTE(__LINE__); }
                    retake_ok = state_cas(pc, w, swith(w, kInUse));
                    cur_word = swith(w, kInUse);
                }
                rec(kEvAcq, cur);
            }
            pf_add(pfBuRetake, now() - tc1);
            const bool stop = C[0] >= P[K - 1];
            bool swap = false;
            if (stop) {
                count(cEarlyStops);
            } else if (elide && !needs_merge_full<Key, K>(C, P)) {
                count(cElided);
                swap = true;  // C < P entirely: parent takes C, the slot takes P
            } else {
                cta_merge_full_bt<Key, K, T>(C, P, buf(ni), buf(si));
                count(cMerges);
            }
            if (!stop) count(cVisits);
            __syncthreads();
            if (leader() && !retake_ok) atomicOr(&hdr->error_flags, (unsigned long long)kErrRetake);
            // the slot's final batch goes to HBM now
            if (stop) {
                if (!cur_written) cta_store<Key, T>(node(cur), C, K);
            } else {
                cta_store<Key, T>(node(cur), swap ? P : buf(si), K);
            }
            __syncthreads();
            pf_lv(2, parent, now() - tc1);
            if (threadIdx.x == kRelLane) lane_unlock(cur);
            if (stop) {
                if (leader()) lane_unlock(parent);  // parent batch unchanged
                if (parent == 1) {
                    pf_add(pfClimbRoot, now() - t_rg);
                    pf_add(pfClimbRootN, 1);
                }
                pf_add(pfInsRest, now() - t3);
                return;
            }
            // carry the parent's new batch up; it is written when released
            if (!swap) {
                const int t = ci;
                ci = ni;
                ni = t;
            }
            cur_written = false;
            cur = parent;
            cur_word = parent_word;
        }
        cta_store<Key, T>(node(1), buf(ci), K);
        __syncthreads();
        if (leader()) lane_unlock(1);
        pf_add(pfClimbRoot, now() - t_rg);
        pf_add(pfClimbRootN, 1);
        pf_add(pfInsRest, now() - t3);
    }

    // ============================================================ delete ==
    // Claims the children of `cur` (acquire_child, heap.cpp:547-585) with
    // lanes 0 and 1 and loads their keys into L/R in the same round trip as
    // the claiming CAS.  TARGET/MARKED children are frozen empty (skipped);
    // INSHOLD children are taken over and released as DELMOD.  Sets
    // sh->lk/rk and sh->lrel/rrel.  Ends with a barrier.
    // The calling thread group is threads [base, base + nthr) with barrier id
    // `bar` (0 = the whole CTA, nthr = T).
    __device__ void acquire_children(unsigned long long cur, Key* L, Key* R, uint32_t base = 0,
                                     uint32_t nthr = T, uint32_t bar = 0) {
        const uint32_t gt = threadIdx.x - base;
        uint32_t pending = 3u;
        if (gt < 2) {
            if (gt == 0) {
                sh->lk = 0;
                sh->lrel = kAvail;
            } else {
                sh->rk = 0;
                sh->rrel = kAvail;
            }
        }
        const unsigned long long t = now();
        for (;;) {
            if (gt < 2 && ((pending >> gt) & 1u)) {
                const unsigned long long slot = 2 * cur + gt;
                uint32_t claim = 0, w = 0;
                if (slot <= hv.slot_count) {
                    uint32_t* p = st(slot);
                    Backoff b(&hdr->error_flags);
                    for (;;) {
                        w = state_load(p);
                        const uint32_t s = sget(w);
                        if (s == kAvail || s == kInsHold || s == kDelMod) {
                            claim = 1;
                            break;
                        }
                        if (s == kTarget || s == kMarked) break;  // frozen empty
                        { b.pause(); BH_WAIT_NOTE(__LINE__); BH_WAIT_NOTE2(slot, w); }
                    }
                }
                sh->claim[gt] = claim;
                sh->cw[gt] = w;
            }
            grp_sync(bar, nthr);
            const uint32_t cl = ((pending & 1u) && sh->claim[0]) | (((pending & 2u) && sh->claim[1]) << 1);
            // the claim CAS goes out first and relaxed, so the key loads below
            // travel in the same round trip (the acquire was the poll)
            uint32_t ok = 0;
            if (gt < 2 && ((cl >> gt) & 1u)) {
                const unsigned long long slot = 2 * cur + gt;
                const uint32_t w = sh->cw[gt];
                ok = state_cas_relaxed(st(slot), w, swith(w, kInUse));
                if (ok) BH_OWN(slot);
            }
            if (cl & 1u) grp_load<Key>(L, node(2 * cur), K, gt, nthr);
            if (cl & 2u) grp_load<Key>(R, node(2 * cur + 1), K, gt, nthr);
            if (gt < 2 && ((cl >> gt) & 1u)) {
                const unsigned long long slot = 2 * cur + gt;
                const uint32_t w = sh->cw[gt];
                sh->ok[gt] = ok;
                if (ok) {
                    rec_lane(kEvAcq, slot);
                    const uint32_t rel = sget(w) == kInsHold ? kDelMod : kAvail;
                    if (gt == 0) {
                        sh->lk = 1;
                        sh->lrel = rel;
                    } else {
                        sh->rk = 1;
                        sh->rrel = rel;
                    }
                }
            }
            grp_sync(bar, nthr);
            uint32_t still = 0;
            if ((cl & 1u) && !sh->ok[0]) still |= 1u;
            if ((cl & 2u) && !sh->ok[1]) still |= 2u;
            pending = still;
            if (!pending) break;
        }
        pf_add(pfChildWait, now() - t);
    }

    // refill_root_from(last) (heap.cpp:467-531), first half.  Leader only.
    // kTake: the last node is claimable from the observed word sh->cw[2]
    // (the caller CASes it while the CTA loads its keys); AVAIL/DELMOD
    // release as AVAIL, an INSHOLD in-flight batch releases as DELMOD.
    // kCoop (TD): TARGET -> MARKED, then wait until the inserter has shipped
    // its batch into the root and set the target AVAIL.
    enum { kTake = 1, kCoop = 2 };
    __device__ void lane_poll_last(unsigned long long last) {
        uint32_t* p = st(last);
        Backoff b(&hdr->error_flags);
        for (;;) {
            const uint32_t w = state_load(p);
            const uint32_t s = sget(w);
            if (s == kAvail || s == kDelMod || s == kInsHold) {
                sh->cw[2] = w;
                sh->act = kTake;
                sh->lastrel = s == kInsHold ? kDelMod : kAvail;
                return;
            }
            if (s == kTarget && state_cas(p, w, swith(w, kMarked))) {
                Backoff wb(&hdr->error_flags);
                while (sget(state_load(p)) != kAvail) { wb.pause(); BH_WAIT_NOTE(__LINE__); }
                sh->act = kCoop;
                return;
            }
            { b.pause(); BH_WAIT_NOTE(__LINE__); }
        }
    }

    // refill_root_from(last), claim + copy + blank + release, by threads
    // [base, base + nthr) with barrier `bar`.  The refill batch lands in dst.
    // `pre`: a state word of `last` observed (acquire) earlier by this CTA;
    // a claim from it skips the first poll (the CAS fails if it changed).
    __device__ void refill_last(unsigned long long last, Key* dst, uint32_t base, uint32_t nthr, uint32_t bar,
                                uint32_t pre = 0xFFFFFFFFu) {
        const uint32_t gt = threadIdx.x - base;
        for (;;) {
            if (gt == 0) {
                const uint32_t ps = sget(pre);
                if (ps == kAvail || ps == kDelMod) {
                    sh->cw[2] = pre;
                    sh->act = kTake;
                    sh->lastrel = kAvail;
                } else {
                    lane_poll_last(last);
                }
                pre = 0xFFFFFFFFu;
            }
            grp_sync(bar, nthr);
            const uint32_t act = sh->act;
            uint32_t ok = 0;
            if (act == kTake && gt == 0) {
                const uint32_t w = sh->cw[2];
                ok = state_cas_relaxed(st(last), w, swith(w, kInUse));
                if (ok) BH_OWN(last);
            }
            grp_load<Key>(dst, node(act == kTake ? last : 1), K, gt, nthr);
            if (act == kCoop) {
                grp_sync(bar, nthr);
                return;
            }
            if (gt == 0) {
                sh->ok[2] = ok;
                if (ok) rec_lane(kEvAcqRefill, last);
            }
            grp_sync(bar, nthr);
            if (sh->ok[2]) {
                grp_fill_max<Key>(node(last), K, gt, nthr);
                grp_sync(bar, nthr);
                if (gt == 0) lane_unlock(last, sh->lastrel);
                return;
            }
        }
    }

    // ================================================== delete serving ==
    // Flat combining of deletes in the root queue lock (TD and BU heaps).  In
    // BU heaps the server's own op passed the phase gate (gate_try, phase =
    // heapify, not closing) and the ops it serves are admitted under that
    // pass (deleters + 1 each, below) without their own gate_try: the gate
    // cannot close during the hold, because closing it takes the root lock,
    // and the hold serves only the contiguous run of delete tickets queued
    // ahead in the FIFO root queue, so a climber that arrives waits for at
    // most those, then closes the phase as usual.
    // A delete holding the root with deletes queued behind it keeps
    // the root and nodes 2-3 (claimed, in shared memory) and runs, for its own
    // op and then each queued delete in ticket order, the reference's
    // delete_min through levels 0 and 1: root result, refill from the last
    // node, the level-0 and level-1 heapify steps (same merges, elisions, hi/lo
    // choices and counters as heapify_down).  The heapify below level 1 --
    // the carried batch and the claimed level-2 node -- is handed to the CTA
    // of the next queued delete (through `mailbox` and its queue slot line),
    // which is woken with it instead of the lock; the last continuation stays
    // with the server.  Each op linearizes at its root step inside this root
    // hold, in queue order, as its own root step would; levels 0-1 pass from
    // one op to the next without a hand-off between SMs, which removes the
    // two-step chain of section 6 from the top of the heap.
    //
    // Releases of an op's level-2 nodes and the hand-off flag of its
    // continuation are deferred to the start of the next op and issued by one
    // lane (kPubLane, outside the refill group) behind a single fence.
    // Deadlock freedom as in the reference: the server waits on a claim only
    // for hi1's children; its refill beside that claim never waits while it
    // holds the last node, and the level-2 nodes of the previous op are
    // released by kPubLane, which waits on nothing; so across the wait the
    // server holds only nodes 1-3, which no other op waits for while holding
    // anything.
    static constexpr unsigned long long kServeMin = 64;  // last node stays below level 5
    static constexpr uint32_t kRefBase = T >= 256 ? 64 : 32;  // refill group: [kRefBase, T/2)
    static constexpr uint32_t kHalfT = T / 2;
    static constexpr uint32_t kPubLane = T >= 256 ? 32 : 1;  // outside the refill group
    // warp 0 claims hi1's children at the op's start (needs warp 1 for kPubLane)
    static constexpr bool kEarlyClaim = T >= 256;

    __device__ __forceinline__ Key* mbox(unsigned long long t) const {
        return static_cast<Key*>(hv.mailbox) + (t % kRootQueue) * (unsigned long long)K;
    }

    // Leader or kPubLane: is ticket t a delete that posted a serve request?
    // The launch, op index and result offset (words 12-13, 2-3, 4-5) load in
    // one round trip after the request word's acquire.
    __device__ bool waiting_delete(unsigned long long t, unsigned long long& op, unsigned long long* off = nullptr) {
        uint32_t* f = qline(t);
        if (state_load(f + 11) != (((uint32_t)t << 1) | 1u)) return false;
        const unsigned long long launch = ld_cg_u64(reinterpret_cast<const unsigned long long*>(f + 12));
        const unsigned long long o = ld_cg_u64(reinterpret_cast<const unsigned long long*>(f + 2));
        const unsigned long long of = ld_cg_u64(reinterpret_cast<const unsigned long long*>(f + 4));
        if (launch != (unsigned long long)rv.ticket) return false;  // a delete of another launch: granted normally
        op = o;
        if (off) *off = of;
        return true;
    }

    // op = ~0: a release not logged (nodes 2-3 at the end of a hold: each
    // served op logged its own spans of them)
    __device__ __forceinline__ void pend(unsigned long long slot, uint32_t rel, unsigned long long op = 0) {
        if (threadIdx.x == kPubLane) {
            sh->pd.slot[sh->pd.n] = slot;
            sh->pd.op[sh->pd.n] = op == ~0ull ? ~0ull : cur_op;
            sh->pd.rel[sh->pd.n] = rel;
            ++sh->pd.n;
        }
    }

    // kPubLane: the previous op's releases, one fence for all of them.  The
    // fence (fence.acq_rel.gpu, cumulative over the CTA's writes ordered
    // before it by the barriers) publishes the mailbox batch, qline word 14
    // and the released nodes' keys; every release after it is relaxed.  (A
    // red.release is a release for its own location only, not a fence.)
    __device__ void sv_flush(SvPending& pd) {
        if (pd.pub && record)  // the op the woken CTA continues, for its events
            st_cg_u64(reinterpret_cast<unsigned long long*>(qline(pd.pub) + 14), pd.pubop);
        if (pd.n || pd.pub) __threadfence();
        for (uint32_t i = 0; i < pd.n; ++i) {
            if (record && pd.op[i] != ~0ull) rec_for(pd.op[i], kEvRel, pd.slot[i]);
            state_release_relaxed(st(pd.slot[i]), kInUse, pd.rel[i]);
        }
        if (pd.pub) {
            const unsigned long long w = ((unsigned long long)pd.pubw << 32) | (((uint32_t)pd.pub << 1) | 1u);
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(qline(pd.pub)), "l"(w) : "memory");
        }
        pd.n = 0;
        pd.pub = 0;
    }

    // Two independent half merges, side by side on the two thread groups when
    // they fit (HalfShape::kPair), else one after the other.  No barrier.
    template <bool S1, bool S2, bool G2 = false>
    __device__ __forceinline__ void two_halves(const Key* A1, const Key* B1, Key* o1, bool do1, const Key* A2,
                                               const Key* B2, Key* o2, bool do2) {
        constexpr int kW = T / 32;
        const uint32_t w = threadIdx.x >> 5;
        if constexpr (kW >= 2) {
            constexpr int kH = kW / 2;
            if (w < (uint32_t)kH) {
                if (do1) grp_merge_half<Key, K, kH, S1, false>(A1, B1, o1, w);
            } else if (w < 2u * kH) {
                if (do2) grp_merge_half<Key, K, kH, S2, G2>(A2, B2, o2, w - kH);
            }
        } else {
            if (do1) grp_merge_half<Key, K, 1, S1, false>(A1, B1, o1, 0);
            if (do2) grp_merge_half<Key, K, 1, S2, G2>(A2, B2, o2, 0);
        }
    }

    // One delete (ticket t) through levels 0 and 1.  Buffers n1/n2/n3 hold
    // nodes 1-3 (in and out).  Returns the continuation node (0 = heapify
    // done) and its release state; its carried batch is in mbox(t + 1) when
    // sh->serve (the next ticket is served next), else in buf(cbuf).  pd:
    // releases due (in) / deferred by this op (out).  Schedule (8 half
    // merges, two at a time):
    //   split  refill (claim, copy, blank) || H0, claim hi1's children, lo0
    //   r1     new root || carried        (halves of merge(refill, H0))
    //   r2     H1 || lo2 -> HBM           (halves of merge(L2, R2))
    //   r3     new hi1 || next carried    (halves of merge(carried, H1))
    __device__ unsigned long long serve_one(unsigned long long opi, unsigned long long off, unsigned long long seq,
                                            unsigned long long nodes, unsigned long long t, int& n1, int& n2,
                                            int& n3, int& cbuf, uint32_t& crel, uint32_t pre_w) {
        const unsigned long long ts0 = now();
        const uint32_t jj = sv_j;  // the op's index in the hold (timeline)
        if (leader()) tl(jj, 0);
        Key* out = static_cast<Key*>(rv.out_pool) + off;
        count(cDeletes);
        if (leader() && buf(n1)[K - 1] == kMaxKey)
            atomicOr(&hdr->error_flags, (unsigned long long)kErrSentinelEscaped);
        status(opi, BH_OK, K, seq);
        if (threadIdx.x >= 8 && threadIdx.x < 8 + kRefillAhead && nodes > threadIdx.x - 8 + 5) {
            const unsigned long long slot = slot_for_rank(nodes - 1 - (threadIdx.x - 8));
            const char* a = reinterpret_cast<const char*>(node(slot));
            for (uint32_t off = 0; off < kNodeBytes; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a + off));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(st(slot)));
        }
        uint32_t used = (1u << n1) | (1u << n2) | (1u << n3);
        auto alloc = [&]() {
            const int b = __ffs(~used) - 1;
            used |= 1u << b;
            return b;
        };
        const Key* L = buf(n2);
        const Key* R = buf(n3);
        // level-0 children decision (independent of the refill)
        const bool lempty = L[0] == kMaxKey, rempty = R[0] == kMaxKey;
        bool hi_left, mc0 = false, el0 = false;
        if (lempty) {
            hi_left = false;
        } else if (rempty) {
            hi_left = true;
        } else if (elide && !needs_merge_full<Key, K>(L, R)) {
            el0 = true;
            hi_left = L[K - 1] <= R[0];  // tie fix of heap.cpp:628-636
        } else {
            hi_left = !(L[K - 1] > R[K - 1]);
            mc0 = true;
        }
        const int rf = alloc(), l2 = alloc(), r2 = alloc();
        const int h0 = mc0 ? alloc() : -1;
        const int nlo = mc0 ? alloc() : (hi_left ? n3 : n2);  // the lo child's new batch
        const unsigned long long hi1 = hi_left ? 2 : 3;
        const unsigned long long c2l = 2 * hi1, c2r = 2 * hi1 + 1;
        const unsigned long long last = slot_for_rank(nodes);
        // split: refill (claim, copy, blank, release the last node) ||
        // H0 and lo0, then the claim of hi1's children.  Warps below kRefBase
        // stay out of both groups: the leader's bookkeeping and kPubLane's
        // flush of the previous op + next-waiter lookup run beside them.
        if (threadIdx.x < 32 && kEarlyClaim) {
            // warp 0: hi1's children (level 2), claimed and loaded at the
            // op's start beside H0 || lo0 and the refill (hi1 is known from
            // nodes 2-3 alone); the one claim the server may wait on
            const unsigned long long tc = now();
            acquire_children(hi1, buf(l2), buf(r2), 0, 32, 3);
            if (threadIdx.x == 0) tl(jj, 5);
            if (prof && threadIdx.x == 0) atomicAdd(&hv.prof[pfSvClaim], now() - tc);
        } else if (threadIdx.x < kRefBase) {
            // (a look-up beside the flush instead of after it -- three lanes,
            // three chains -- hung mixed insert/delete runs with serving at
            // full size, tools/gpu/bisect_mixed.sh; the order below is the
            // tested one)
            if (threadIdx.x == kPubLane) {
                sv_flush(sh->pd);
                tl(jj, 1);
                unsigned long long nop = 0;
                const bool more = nodes - 1 >= kServeMin && waiting_delete(t + 1, nop);
                sh->serve = more;
                sh->op_next = nop;
                if (more) {
                    sh->off_next = rv.ops[nop].offset;
                    sh->next_w = state_load(st(slot_for_rank(nodes - 1)));  // the next op's refill
                }
                tl(jj, 2);
            }
        } else if (threadIdx.x < kHalfT) {
            // released here, before the server waits on any claim (below)
            refill_last(last, buf(rf), kRefBase, kHalfT - kRefBase, 1, pre_w);
            // the refill batch usually moves down levels 0-1 unchanged and is
            // then the carried batch this op hands to the next ticket: into
            // its mailbox now, long before the next op's publishing fence
            // (overwritten in round 3 when it is not; unread when the hold
            // ends)
            grp_store<Key>(mbox(t + 1), buf(rf), K, threadIdx.x - kRefBase, kHalfT - kRefBase);
            if (threadIdx.x == kRefBase) tl(jj, 3);
            if (prof && threadIdx.x == kRefBase) atomicAdd(&hv.prof[pfSvA], now() - ts0);
        } else {
            // both halves of merge(L, R): H0 and the lo child's new batch,
            // then hi1's children: the one claim the server may wait on (for
            // the continuation of the previous op on the same side), issued
            // last.  The refill beside it never waits while holding the last
            // node, so nothing but nodes 1-3 is held across this wait.
            if (mc0) {
                // two quarter groups side by side (T >= 128 here)
                constexpr int kQ = T >= 128 ? T / 128 : 1;
                const uint32_t bw = (threadIdx.x - kHalfT) >> 5;
                if (bw < (uint32_t)kQ) grp_merge_half<Key, K, kQ, false, false>(L, R, buf(h0), bw);
                else grp_merge_half<Key, K, kQ, true, false>(L, R, buf(nlo), bw - kQ);
            }
            if (threadIdx.x == kHalfT) tl(jj, 4);
            if (prof && threadIdx.x == kHalfT) atomicAdd(&hv.prof[pfSvB], now() - ts0);
            if constexpr (!kEarlyClaim) {
                const unsigned long long tc = now();
                acquire_children(hi1, buf(l2), buf(r2), kHalfT, kHalfT, 2);
                if (threadIdx.x == kHalfT) tl(jj, 5);
                if (prof && threadIdx.x == kHalfT) atomicAdd(&hv.prof[pfSvClaim], now() - tc);
            }
        }
        // (timeline stamps are taken where a warp *reaches* a barrier: a
        // clock read right after BAR.SYNC.DEFER_BLOCKING issues before the
        // warp blocks, tools/microbench/mb_barmix.cu)
        if (threadIdx.x == kHalfT + 32) tl(jj, 6);
        __syncthreads();
        // the result (the root's k keys), written after the split: stores
        // issued at the op's start would sit in front of kPubLane's fence,
        // which publishes the previous op's continuation (the chain)
        {
            const uint4* sv = reinterpret_cast<const uint4*>(buf(n1));
            uint4* gv = reinterpret_cast<uint4*>(out);
            for (uint32_t i = threadIdx.x; i < kNodeBytes / 16; i += T) __stcg(gv + i, sv[i]);
        }
        const unsigned long long ts1 = now();
        pf_add(pfSvSplit, ts1 - ts0);
        const bool handoff = sh->serve != 0;
        const Key* RF = buf(rf);

        // ---- level 0: cur = the refill ----
        const Key cmax = RF[K - 1];
        bool stop0 = lempty && rempty;
        if (!stop0 && cmax <= (lempty ? kMaxKey : L[0]) && cmax <= (rempty ? kMaxKey : R[0])) {
            count(cEarlyStops);
            stop0 = true;
        }
        const uint32_t lk2 = sh->lk, rk2 = sh->rk, lrel2 = sh->lrel, rrel2 = sh->rrel;
        if (stop0) {  // the refill is the new root, levels 1-2 unchanged
            if (lk2) pend(c2l, lrel2);
            if (rk2) pend(c2r, rrel2);
            n1 = rf;
            return 0;
        }
        if (mc0) count(cMerges);
        else if (el0) count(cElided);
        const int hd0 = mc0 ? h0 : (hi_left ? n2 : n3);
        const bool mcur0 = !(elide && !needs_merge_full<Key, K>(RF, buf(hd0)));
        count(mcur0 ? cMerges : cElided);
        count(cVisits);
        // live: rf, hd0, nlo, l2, r2
        used = (1u << rf) | (1u << hd0) | (1u << nlo) | (1u << l2) | (1u << r2);
        int nr, ca;
        if (mcur0) {
            nr = alloc();
            ca = alloc();
            two_halves<false, true>(RF, buf(hd0), buf(nr), true, RF, buf(hd0), buf(ca), true);
        } else {  // full inversion: the hi batch moves up, the refill goes down
            nr = hd0;
            ca = rf;
        }
        pf_add(pfSvR1, now() - ts1);
        // (a CTA barrier costs ~250-450 cycles here: none when the round
        // wrote nothing -- the refill moved down unchanged)
        if (mcur0) __syncthreads();
        if (leader()) tl(jj, 7);
        const unsigned long long ts2 = now();

        // ---- level 1: cur = carried batch at hi1, children claimed above ----
        used = (1u << nr) | (1u << nlo) | (1u << ca) | (1u << l2) | (1u << r2);
        const Key* L2 = buf(l2);
        const Key* R2 = buf(r2);
        const Key* CA = buf(ca);
        const bool le2 = !lk2 || L2[0] == kMaxKey, re2 = !rk2 || R2[0] == kMaxKey;
        const Key cmax1 = CA[K - 1];
        bool stop1 = le2 && re2;
        if (!stop1 && cmax1 <= (le2 ? kMaxKey : L2[0]) && cmax1 <= (re2 ? kMaxKey : R2[0])) {
            count(cEarlyStops);
            stop1 = true;
        }
        unsigned long long cont = 0;
        int nhi;
        if (stop1) {
            nhi = ca;
            if (lk2) pend(c2l, lrel2);
            if (rk2) pend(c2r, rrel2);
        } else {
            bool hl1, mc1 = false;
            if (le2) {
                hl1 = false;
            } else if (re2) {
                hl1 = true;
            } else if (elide && !needs_merge_full<Key, K>(L2, R2)) {
                count(cElided);
                hl1 = L2[K - 1] <= R2[0];
            } else {
                hl1 = !(L2[K - 1] > R2[K - 1]);
                mc1 = true;
                count(cMerges);
            }
            const unsigned long long hi2 = hl1 ? c2l : c2r, lo2 = hl1 ? c2r : c2l;
            const uint32_t lo2_locked = hl1 ? rk2 : lk2;
            const uint32_t hi2_rel = hl1 ? lrel2 : rrel2, lo2_rel = hl1 ? rrel2 : lrel2;
            const int h1 = mc1 ? alloc() : -1;
            if (mc1) {
                // H1 || lo2's batch (second half of merge(L2, R2)) -> HBM
                two_halves<false, true, true>(L2, R2, buf(h1), true, L2, R2, node(lo2), true);
                __syncthreads();
            }
            const unsigned long long ts3 = now();
            if (leader()) tl(jj, 8);
            pf_add(pfSvR2, ts3 - ts2);
            const int hd1 = mc1 ? h1 : (hl1 ? l2 : r2);
            const bool mcur1 = !(elide && !needs_merge_full<Key, K>(CA, buf(hd1)));
            count(mcur1 ? cMerges : cElided);
            count(cVisits);
            // the carried batch goes straight to the next ticket's mailbox
            // when that op is served next, else it stays here
            if (mcur1) {
                nhi = alloc();
                cbuf = alloc();
                if (handoff)
                    two_halves<false, true, true>(CA, buf(hd1), buf(nhi), true, CA, buf(hd1), mbox(t + 1), true);
                else
                    two_halves<false, true>(CA, buf(hd1), buf(nhi), true, CA, buf(hd1), buf(cbuf), true);
            } else {
                nhi = hd1;
                cbuf = ca;
                if (handoff && ca != rf) cta_store<Key, T>(mbox(t + 1), CA, K);
            }
            if (lo2_locked) pend(lo2, lo2_rel);  // merged above, or unchanged
            cont = hi2;
            crel = hi2_rel;
            pf_add(pfSvR3, now() - ts3);
        }
        // (no barrier here: serve_deletes' loop barrier, before the next op
        // or the write-back, orders this round's writes)
        if (leader()) tl(jj, 9);
        n1 = nr;
        if (hi1 == 2) {
            n2 = nhi;
            n3 = nlo;
        } else {
            n3 = nhi;
            n2 = nlo;
        }
        return cont;
    }

    // Root held (ticket sh->root_tk), gate passed, buf(0) = root batch,
    // partial buffer empty, the next ticket a waiting delete.
    __device__ void serve_deletes(unsigned long long opi, unsigned long long seq, unsigned long long nodes) {
        int n1 = 0, n2 = 1, n3 = 2;
        acquire_children(1, buf(n2), buf(n3));
        const uint32_t rel2 = sh->lrel, rel3 = sh->rrel;
        unsigned long long t = sh->root_tk, op = opi, served = 0, off = rv.ops[opi].offset;
        uint32_t pre_w = 0xFFFFFFFFu;
        int cbuf = -1;
        uint32_t crel = kAvail;
        unsigned long long cont = 0;
        if (threadIdx.x == kPubLane) {
            sh->pd.n = 0;
            sh->pd.pub = 0;
        }
        sv_j = 0;
        if (prof && threadIdx.x == 0)
            for (uint32_t i = 0; i < kTlSmemOps * 24u; ++i) sh->tl[i] = 0;
        __syncthreads();

        for (;; ++sv_j) {
            cur_op = op;  // the lock events of this op's top levels are its own
            if (record && served && leader()) {  // the first op holds 1-3 already
                rec(kEvAcq, 1);
                rec(kEvAcq, 2);
                rec(kEvAcq, 3);
            }
            cont = serve_one(op, off, seq, nodes, t, n1, n2, n3, cbuf, crel, pre_w);
            if (record && leader()) {
                rec(kEvRel, 2);
                rec(kEvRel, 3);
                rec(kEvRel, 1);
            }
            const unsigned long long tn = now();
            ++seq;
            --nodes;
            const bool more = sh->serve != 0;
            const unsigned long long nop = sh->op_next;
            const unsigned long long noff = sh->off_next;
            pre_w = sh->next_w;  // the next op's refill word, observed in this op
            __syncthreads();  // everyone has read sh->serve / op_next
            if (leader()) tl(sv_j, 10);
            if (!more) break;
            // the waiter of ticket t+1 takes this op's continuation (its
            // carried batch is in mbox(t+1)); its own op is served next.  The
            // flag goes out with the next op's flush.
            if (threadIdx.x == kPubLane) {
                if (hv.variant == BH_BU) atomicAdd(&hdr->deleters, 1ull);  // op t+1 is in the delete phase
                sh->pd.pub = t + 1;
                sh->pd.pubw = (uint32_t)cont | (crel == kDelMod ? 0x80000000u : 0u);
                sh->pd.pubop = op;
            }
            op = nop;
            off = noff;
            ++t;
            ++served;
            pf_add(pfSvNext, now() - tn);
        }
        if (prof)  // the timeline (first hold of the run only)
            for (uint32_t i = threadIdx.x; i < kTlSmemOps * 24u; i += T)
                if (sh->tl[i]) atomicCAS(&hv.prof[kTlBase + (i / 24u) * 32u + i % 24u], 0ull, sh->tl[i]);
        // write the top levels back, then release everything and the root
        cta_store<Key, T>(node(1), buf(n1), K);
        cta_store<Key, T>(node(2), buf(n2), K);
        cta_store<Key, T>(node(3), buf(n3), K);
        if (leader()) {
            st_cg_u64(&hdr->node_count, nodes);
            st_cg_u64(&hdr->delete_count, seq);
        }
        __syncthreads();
        pend(2, rel2, ~0ull);
        pend(3, rel3, ~0ull);
        if (threadIdx.x == kPubLane) {
            sv_flush(sh->pd);  // its fence also orders nodes 1-3 and the header
            sh->root_tk = t;
            state_store_relaxed(qline(t + 1), (uint32_t)(t + 1) << 1);  // root_unlock
        }
        pf_add(pfDelServed, served);
        pf_add(pfDelServeHolds, served ? 1 : 0);
        cur_op = op;  // the last op served: its continuation stays here
        if (cont) heapify_down(cbuf, 0, false, cont, crel);
        rec(kEvRes, 0);
        if (hv.variant == BH_BU && leader()) gate_leave(false);
    }

    // ========================================= three-level delete server ==
    // serve3: delete serving (flat combining of deletes in the root queue
    // lock, see serve_deletes) with levels 0-2 -- nodes 1-7 -- held in shared
    // memory, and the work of one op split over warp roles that hand off
    // through mbarriers instead of CTA-wide barriers:
    //   warp 0      control: result of the op (the root batch), the previous
    //               op's level-3 releases and continuation hand-off (one
    //               fence), look-ups of the next two tickets, refill requests,
    //               counters and the event log;
    //   warp 1      claims hi2's children (level 3, the one place the server
    //               waits on another CTA) and loads them;
    //   warps 2-13  the merges, in four rounds: H0 || H1 || lo0 || lo1;
    //               new root || carried 1; new hi1 || carried 2 || H2 || lo2;
    //               new hi2 || carried 3 (to the next ticket's mailbox) ||
    //               the lo level-3 child back to HBM;
    //   warps 14-15 refills, one op each in turn, one op AHEAD: the refill
    //               source of op j+1 (the last node after op j) is claimed,
    //               copied, blanked and released while op j is merged.
    // Every op still runs the reference's delete_min (heap.cpp:411-667):
    // the same root result, refill source, per-level early stop, elisions,
    // hi/lo choices (with the tie fix) and counters as heapify_down; levels
    // 0-2 of op j and the refill of op j+1 touch disjoint nodes (the refill
    // source is at level >= 5), so running them side by side is equivalent to
    // running them in order.  The path through levels 0-2 depends only on
    // the children's batches, so warp 1 knows at the op's start which
    // level-3 nodes the op needs.  Deadlock freedom as for serve_deletes:
    // the server waits on other CTAs only in warp 1's level-3 claims and in
    // the refill warps' claim of the last node; the refill warps hold the
    // last node only to copy and blank it; the continuation of the previous
    // op is published by warp 0, which waits on nothing but this CTA's own
    // merges; across the waits the server holds nodes 1-7, which nobody
    // waits for while holding anything.
    static constexpr bool kS3 = Serve3Cfg<Key, K, T>::kOn;
    static constexpr uint32_t kS3OpThreads = 416;     // warps 0 and 2-13
    static constexpr uint32_t kS3MergeThreads = 384;  // warps 2-13
    static constexpr uint32_t kS3BarOp = 5, kS3BarMerge = 6;
    static constexpr uint32_t kS3MergeLeader = 64;    // lane 0 of warp 2
    static constexpr uint32_t kVecs = kNodeBytes / 16;

    __device__ __forceinline__ void warp_load_node(Key* s, const Key* g) const {
        const uint32_t lane = threadIdx.x & 31u;
        const uint4* gv = reinterpret_cast<const uint4*>(g);
        uint4* sv = reinterpret_cast<uint4*>(s);
#pragma unroll 8
        for (uint32_t i = lane; i < kVecs; i += 32) sv[i] = __ldcg(gv + i);
    }
    __device__ __forceinline__ void warp_store_node(Key* g, const Key* s) const {
        const uint32_t lane = threadIdx.x & 31u;
        uint4* gv = reinterpret_cast<uint4*>(g);
        const uint4* sv = reinterpret_cast<const uint4*>(s);
#pragma unroll 8
        for (uint32_t i = lane; i < kVecs; i += 32) __stcg(gv + i, sv[i]);
    }
    __device__ __forceinline__ void warp_fill_node(Key* g) const {
        const uint32_t lane = threadIdx.x & 31u;
        uint4 f;
        f.x = f.y = f.z = f.w = 0xFFFFFFFFu;
        uint4* gv = reinterpret_cast<uint4*>(g);
#pragma unroll 8
        for (uint32_t i = lane; i < kVecs; i += 32) __stcg(gv + i, f);
    }

    // hi/lo of two non-empty sibling batches (heap.cpp:628-652, tie fix)
    __device__ __forceinline__ void s3_children(const Key* L, const Key* R, bool& mc, bool& el, bool& hl) const {
        if (elide && !needs_merge_full<Key, K>(L, R)) {
            el = true;
            mc = false;
            hl = L[K - 1] <= R[0];
        } else {
            el = false;
            mc = true;
            hl = !(L[K - 1] > R[K - 1]);
        }
    }

    // One warp: acquire_child (heap.cpp:547-585) of both children of `cur`,
    // lanes 0/1 polling and claiming, the keys loaded by the whole warp in the
    // claim's round trip.  Returns locked bits (1 = left, 2 = right); rel
    // states in lrel/rrel (DELMOD for an INSHOLD take-over).
    // `guess` (lanes 0/1): a claimable word of the child, observed by an
    // acquire load of this warp after the node's last release or produced by
    // this CTA's own release (0xFFFFFFFF = none): the first CAS goes out with
    // it, with no poll before it; a changed word fails the CAS.
    __device__ uint32_t warp_claim_children(unsigned long long cur, Key* L, Key* R, uint32_t& lrel, uint32_t& rrel,
                                            uint32_t guess, uint32_t& claimed_w, uint32_t* ntries = nullptr) {
        const uint32_t lane = threadIdx.x & 31u;
        uint32_t pending = 3u, locked = 0;
        lrel = rrel = kAvail;
        while (pending) {
            if (ntries) ++*ntries;
            uint32_t claim = 0, w = 0;
            const uint32_t gs = sget(guess);
            if (lane < 2 && ((pending >> lane) & 1u)) {
                const unsigned long long slot = 2 * cur + lane;
                if (guess != 0xFFFFFFFFu && (gs == kAvail || gs == kDelMod || gs == kInsHold)) {
                    claim = 1;
                    w = guess;
                } else if (slot <= hv.slot_count) {
                    uint32_t* p = st(slot);
                    Backoff b(&hdr->error_flags);
                    for (;;) {
                        w = state_poll(p);  // relaxed poll + acquire fence (no L1 invalidation per poll)
                        const uint32_t s = sget(w);
                        if (s == kAvail || s == kInsHold || s == kDelMod) {
                            acquire_fence();
                            claim = 1;
                            break;
                        }
                        if (s == kTarget || s == kMarked) break;  // frozen empty
                        b.pause();
                    }
                }
            }
            const uint32_t cl = (__shfl_sync(0xFFFFFFFFu, claim, 0) ? 1u : 0u) |
                                (__shfl_sync(0xFFFFFFFFu, claim, 1) ? 2u : 0u);
            uint32_t ok = 0;
            if (lane < 2 && ((cl >> lane) & 1u)) ok = state_cas_relaxed(st(2 * cur + lane), w, swith(w, kInUse));
            if (cl & 1u) warp_load_node(L, node(2 * cur));
            if (cl & 2u) warp_load_node(R, node(2 * cur + 1));
            const uint32_t okm = (__shfl_sync(0xFFFFFFFFu, ok, 0) ? 1u : 0u) |
                                 (__shfl_sync(0xFFFFFFFFu, ok, 1) ? 2u : 0u);
            const uint32_t w0 = __shfl_sync(0xFFFFFFFFu, w, 0), w1 = __shfl_sync(0xFFFFFFFFu, w, 1);
            if (lane < 2 && ((okm >> lane) & 1u)) rec_lane(kEvAcq, 2 * cur + lane);
            if (okm & 1u) lrel = sget(w0) == kInsHold ? kDelMod : kAvail;
            if (okm & 2u) rrel = sget(w1) == kInsHold ? kDelMod : kAvail;
            if (lane < 2 && ((okm >> lane) & 1u)) claimed_w = swith(w, kInUse);
            locked |= okm;
            pending &= ~((pending & ~cl) | okm);  // frozen empty or claimed: done
            guess = 0xFFFFFFFFu;                  // a failed guess: poll
        }
        __syncwarp();
        return locked;
    }

    // One warp: refill_root_from(last) (heap.cpp:467-531) into dst, then
    // arrive on mb (the batch is in shared memory), then blank the last node
    // and release it.  Never waits while holding the last node.  TD: a
    // TARGET last node is MARKED and the inserter ships its batch into node 1
    // in HBM (ship_to_root, heap.cpp:207-216), read from there.
    // `guess` (lane 0): the last node's word observed by this warp's acquire
    // load after its last release (0xFFFFFFFF = none): CAS it at once.
    __device__ void warp_refill(unsigned long long last, Key* dst, unsigned long long* mb, uint32_t guess,
                                uint32_t jj = ~0u) {
        const uint32_t lane = threadIdx.x & 31u;
        uint32_t* p = st(last);
        for (;;) {
            uint32_t act = 0, w = 0;
            const uint32_t gs = sget(guess);
            if (lane == 0 && guess != 0xFFFFFFFFu && (gs == kAvail || gs == kDelMod || gs == kInsHold)) {
                act = kTake;
                w = guess;
            } else if (lane == 0) {
                Backoff b(&hdr->error_flags);
                for (;;) {
                    w = state_poll(p);
                    const uint32_t s = sget(w);
                    if (s == kAvail || s == kDelMod || s == kInsHold) {
                        acquire_fence();
                        act = kTake;
                        break;
                    }
                    if (s == kTarget && state_cas(p, w, swith(w, kMarked))) {
                        Backoff wb(&hdr->error_flags);
                        while (sget(state_load(p)) != kAvail) wb.pause();
                        act = kCoop;
                        break;
                    }
                    b.pause();
                }
            }
            act = __shfl_sync(0xFFFFFFFFu, act, 0);
            w = __shfl_sync(0xFFFFFFFFu, w, 0);
            uint32_t ok = 0;
            if (act == kTake && lane == 0) ok = state_cas_relaxed(p, w, swith(w, kInUse));
            warp_load_node(dst, node(act == kTake ? last : 1));
            ok = __shfl_sync(0xFFFFFFFFu, ok, 0);
            if (act == kCoop) {
                __syncwarp();
                if (lane == 0) mb_arrive(mb);
                return;
            }
            guess = 0xFFFFFFFFu;
            if (!ok) continue;
            if (lane == 0) rec_lane(kEvAcqRefill, last);
            __syncwarp();
            if (lane == 0) {
                mb_arrive(mb);
                tl(jj, 16);
                if (prof && jj - kTlFirst < kTlSmemOps) sh->tl[(jj - kTlFirst) * 24u + 20] = guess != 0xFFFFFFFFu;
            }
            warp_fill_node(node(last));
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                rec_lane(kEvRel, last);
                state_release_relaxed(p, kInUse, sget(w) == kInsHold ? kDelMod : kAvail);
            }
            return;
        }
    }

    // Claim warp: lanes 0-7 check tickets t0..t0+7 at once (serve_deletes'
    // waiting_delete: a delete of this launch that posted a serve request,
    // its op index and result offset from its queue slot line) and note the
    // confirmed ones in the look-ahead ring; one batch of two round trips
    // covers the next several ops.
    __device__ void s3_lookahead(unsigned long long t0) {
        Sv3Shared& s3 = sh->s3;
        const uint32_t lane = threadIdx.x & 31u;
        if (lane < 8) {
            const unsigned long long x = t0 + lane;
            if (s3.la_tk[x & 7u] != x) {
                uint32_t* f = qline(x);
                // relaxed poll, acquire fence only on a match (acquire loads
                // invalidate L1 and stall the merge warps' shared memory work)
                if (state_poll(f + 11) == (((uint32_t)x << 1) | 1u)) {
                    acquire_fence();
                    const unsigned long long launch = ld_cg_u64(reinterpret_cast<const unsigned long long*>(f + 12));
                    const unsigned long long o = ld_cg_u64(reinterpret_cast<const unsigned long long*>(f + 2));
                    const unsigned long long of = ld_cg_u64(reinterpret_cast<const unsigned long long*>(f + 4));
                    if (launch == (unsigned long long)rv.ticket) {
                        s3.la_op[x & 7u] = o;
                        s3.la_off[x & 7u] = of;
                        __threadfence_block();
                        *reinterpret_cast<volatile unsigned long long*>(&s3.la_tk[x & 7u]) = x;
                    }
                }
            }
        }
        __syncwarp();
    }
    __device__ __forceinline__ bool s3_have(unsigned long long x) const {
        const bool y = *reinterpret_cast<volatile const unsigned long long*>(&sh->s3.la_tk[x & 7u]) == x;
        __threadfence_block();  // the entry's op/offset were written before its tag
        return y;
    }

    // Warp 1 of a three-level server: per op, claims hi2's children (level 3)
    // on the merge leader's request (sent one op ahead); in between, looks
    // ahead in the root queue for the next waiting deletes (the ring).  A
    // claim first CASes the word the server's own release of the node
    // produced (the data is then the server's own), else polls.
    __device__ void s3_claim_loop() {
        Sv3Shared& s3 = sh->s3;
        const uint32_t lane = threadIdx.x & 31u;
        unsigned long long t = sh->root_tk;
        for (uint32_t n = 0;; ++n) {
            for (;;) {
                if (__shfl_sync(0xFFFFFFFFu, (uint32_t)mb_test(&s3.mb_go3, n & 1u), 0)) break;
                bool need = false;
                if (lane < 8) need = s3.la_tk[(t + 1 + lane) & 7u] != t + 1 + lane;
                if (__any_sync(0xFFFFFFFFu, need)) s3_lookahead(t + 1);
                __nanosleep(64);
            }
            const uint32_t hi2 = s3.g3_hi2;
            if (!hi2) break;
            const unsigned long long tc = now();
            t = s3.g3_t;
            cur_op = s3.g3_op;
            const uint32_t jj = s3.g3_j;
            if (lane == 0) tl(jj, 13);
            const uint32_t bL = s3.g3_L, bR = s3.g3_R;
            const uint32_t i0 = 2u * hi2 - 8u;
            uint32_t guess = 0xFFFFFFFFu, lrel, rrel, cw = 0, ntries = 0;
            if (lane < 2) guess = s3.w3pred[i0 + lane];
            const uint32_t lk = warp_claim_children(hi2, buf(bL), buf(bR), lrel, rrel, guess, cw, &ntries);
            if (lane < 2 && ((lk >> lane) & 1u)) s3.w3in[i0 + lane] = cw;
            __syncwarp();
            if (lane == 0) {
                s3.lk3 = lk & 1u;
                s3.rk3 = lk >> 1;
                s3.lrel3 = lrel;
                s3.rrel3 = rrel;
                mb_arrive(&s3.mb_c3);
                tl(jj, 14);
                if (prof && jj - kTlFirst < kTlSmemOps) sh->tl[(jj - kTlFirst) * 24u + 18] = ntries;
            }
            if (prof && lane == 0) atomicAdd(&hv.prof[pf3Claim], now() - tc);
        }
    }

    // Root held (ticket sh->root_tk), gate passed, buf(0) = root batch,
    // partial buffer empty, >= kServeMin nodes, the next ticket a waiting
    // delete of this launch.
    __device__ void serve3(unsigned long long opi, unsigned long long seq, unsigned long long nodes) {
        Sv3Shared& s3 = sh->s3;
        const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
        if (threadIdx.x == 0) {
            mb_init(&s3.mb_go[0], 1);
            mb_init(&s3.mb_go[1], 1);
            mb_init(&s3.mb_rf[0], 1);
            mb_init(&s3.mb_rf[1], 1);
            mb_init(&s3.mb_c3, 1);
            mb_init(&s3.mb_go3, 1);
            mb_init(&s3.mb_rec, 1);
        }
        // ---- hold start: nodes 2..7 into buffers 1..6 (root in buffer 0)
        uint32_t delmod = 0, okall;
        acquire_children(1, buf(1), buf(2));
        okall = sh->lk & sh->rk;
        delmod |= (sh->lrel == kDelMod ? 1u << 2 : 0u) | (sh->rrel == kDelMod ? 1u << 3 : 0u);
        __syncthreads();
        acquire_children(2, buf(3), buf(4));
        okall &= sh->lk & sh->rk;
        delmod |= (sh->lrel == kDelMod ? 1u << 4 : 0u) | (sh->rrel == kDelMod ? 1u << 5 : 0u);
        __syncthreads();
        acquire_children(3, buf(5), buf(6));
        okall &= sh->lk & sh->rk;
        delmod |= (sh->lrel == kDelMod ? 1u << 6 : 0u) | (sh->rrel == kDelMod ? 1u << 7 : 0u);
        if (threadIdx.x == 0) {
            if (!okall) atomicOr(&hdr->error_flags, (unsigned long long)kErrInteriorEmpty);
            s3.w0_done = 0;
            s3.w0_seen = 0;
            if (prof)
                for (uint32_t i = 0; i < kTlSmemOps * 24u; ++i) sh->tl[i] = 0;
            for (int i = 0; i < 8; ++i) {
                s3.la_tk[i] = ~0ull;
                s3.w3pred[i] = 0xFFFFFFFFu;
            }
        }
        __syncthreads();

        if (warp >= 14) {
            // ---- refill warps: one op each in turn
            // (each warp observes its next source -- two ranks lower -- once
            // its refill is done, so the next claim needs no poll)
            const uint32_t g = warp - 14;
            unsigned long long pre_rank = 0;
            uint32_t pre_w = 0xFFFFFFFFu;
            for (uint32_t n = 0;; ++n) {
                // idle until the next request: test + sleep (a try_wait spin
                // would take issue slots from the merge warps of its SMSP)
                while (__shfl_sync(0xFFFFFFFFu, (uint32_t)mb_test(&s3.mb_go[g], n & 1u), 0) == 0) __nanosleep(100);
                const unsigned long long rank = s3.go_last[g];
                if (!rank) break;
                const uint32_t b = s3.go_buf[g];
                const uint32_t jj = s3.go_j[g];
                cur_op = s3.go_op[g];
                const unsigned long long tr = now();
                if (lane == 0) tl(jj, 15);
                warp_refill(slot_for_rank(rank), buf(b), &s3.mb_rf[g], rank == pre_rank ? pre_w : 0xFFFFFFFFu, jj);
                if (lane == 0) tl(jj, 17);
                if (prof && lane == 0) atomicAdd(&hv.prof[pf3Refill], now() - tr);
                pre_rank = rank > 2 ? rank - 2 : 0;
                if (lane == 0 && pre_rank) pre_w = state_load(st(slot_for_rank(pre_rank)));
            }
        } else if (warp == 1) {
            s3_claim_loop();
        } else if (warp == 0) {
            s3_control_loop();
        } else {
            s3_merge_loop(opi, seq, nodes);
        }
        __syncthreads();

        if (prof)  // the timeline (first hold of the run only)
            for (uint32_t i = threadIdx.x; i < kTlSmemOps * 24u; i += T)
                if (sh->tl[i]) atomicCAS(&hv.prof[kTlBase + (i / 24u) * 32u + i % 24u], 0ull, sh->tl[i]);
        // ---- hold end: write the top levels back, release them, the last
        // op's level-3 nodes and the root; run its continuation here
        const Sv3Rec& R = s3.rec[(s3.w0_done - 1u) & 3u];
        const unsigned long long t = R.t;
        const unsigned long long lastop = R.op;
        nodes = sh->nodes;
        seq = R.seq + 1;
        for (int i = 1; i <= 7; ++i) cta_store<Key, T>(node(i), buf(s3.nb_end[i]), K);
        if (leader()) {
            st_cg_u64(&hdr->node_count, nodes);
            st_cg_u64(&hdr->delete_count, seq);
        }
        __syncthreads();
        if (leader()) {
            for (uint32_t i = 0; i < R.nrel; ++i) rec_for(lastop, kEvRel, R.relslot[i]);
            __threadfence();
            for (uint32_t i = 2; i <= 7; ++i) state_release_relaxed(st(i), kInUse, ((delmod >> i) & 1u) ? kDelMod : kAvail);
            for (uint32_t i = 0; i < R.nrel; ++i) state_release_relaxed(st(R.relslot[i]), kInUse, R.relst[i]);
            state_store_relaxed(qline(t + 1), (uint32_t)(t + 1) << 1);  // root_unlock
        }
        cur_op = lastop;
        const unsigned long long cont = R.cont;
        const uint32_t crel = R.crel;
        // the carried batch of the last op's continuation: in shared memory,
        // or in the mailbox of ticket t+1 (no one else reads that slot)
        int cb = (int)R.c3buf;
        if (cont && R.c3buf == 0xFFFFFFFFu) {
            cb = 23;
            cta_load<Key, T>(buf(cb), mbox(t + 1), K);
        }
        __syncthreads();
        if (cont) heapify_down(cb, 0, false, cont, crel);
        rec(kEvRes, 0);
        if (hv.variant == BH_BU && leader()) gate_leave(false);
    }

    // Control warp (warp 0) of a three-level server, one op behind the
    // merges: for each op record (in op order): the result (the root batch
    // before the op), then the hand-off of the op's continuation to the CTA of
    // the next ticket (carried batch into its mailbox if still in shared
    // memory, one fence, the op's level-3 releases, the served flag with the
    // continuation word).  Never waits on another CTA.
    __device__ void s3_control_loop() {
        Sv3Shared& s3 = sh->s3;
        const uint32_t lane = threadIdx.x & 31u;
        for (uint32_t j = 0;; ++j) {
            while (__shfl_sync(0xFFFFFFFFu, (uint32_t)mb_test(&s3.mb_rec, j & 1u), 0) == 0) __nanosleep(32);
            const unsigned long long tc = now();
            if (lane == 0) {
                tl(j, 11);
                s3.w0_seen = j + 1;
            }
            const Sv3Rec& R = s3.rec[j & 3u];
            warp_store_node(static_cast<Key*>(rv.out_pool) + R.off, buf(R.rootbuf));
            if (lane == 0 && buf(R.rootbuf)[K - 1] == kMaxKey)
                atomicOr(&hdr->error_flags, (unsigned long long)kErrSentinelEscaped);
            status(R.op, BH_OK, K, R.seq);
            count(cDeletes);
            count(cMerges, R.cnt_merges);
            count(cElided, R.cnt_elided);
            count(cEarlyStops, R.cnt_early);
            count(cVisits, R.cnt_visits);
            if (!R.last) {
                if (R.cont && R.c3buf != 0xFFFFFFFFu) warp_store_node(mbox(R.t + 1), buf(R.c3buf));
                __syncwarp();
                if (lane == 0) {
                    const unsigned long long pub = R.t + 1;
                    if (record) {
                        for (uint32_t i = 0; i < R.nrel; ++i) rec_for(R.op, kEvRel, R.relslot[i]);
                        st_cg_u64(reinterpret_cast<unsigned long long*>(qline(pub) + 14), R.op);
                    }
                    __threadfence();  // the mailbox batch, the released nodes' keys, word 14
                    for (uint32_t i = 0; i < R.nrel; ++i) state_release_relaxed(st(R.relslot[i]), kInUse, R.relst[i]);
                    if (hv.variant == BH_BU) atomicAdd(&hdr->deleters, 1ull);  // op j+1 is in the delete phase
                    const uint32_t pubw = (uint32_t)R.cont | (R.crel == kDelMod ? 0x80000000u : 0u);
                    const unsigned long long w = ((unsigned long long)pubw << 32) | (((uint32_t)pub << 1) | 1u);
                    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(qline(pub)), "l"(w) : "memory");
                }
            }
            __syncwarp();
            if (lane == 0) {
                tl(j, 12);
                s3.w0_done = j + 1;
            }
            if (prof && lane == 0) atomicAdd(&hv.prof[pf3Ctl], now() - tc);
            if (R.last) break;
        }
    }

    // Warps 2-13 of a three-level server: the op loop.  Every merge thread
    // computes the same decisions, node map and buffer plan; the merge leader
    // sends the requests (level-3 claim, refills), writes the records and
    // decides whether the hold goes on.  Per op, after the refill batch is in:
    //   fast path (no merge of a carried batch at levels 0-1: the refill
    //   batch moves down unchanged, the usual case): round A H0 || lo0 || H1,
    //   round B lo1 || H2 || lo2 (to HBM) once the level-3 children are in,
    //   round C new hi2 || carried 3 only when the refill interleaves H2;
    //   general path: the four rounds of serve_deletes' schedule, one level
    //   deeper.
    // Every merge runs through one inlined call site (instruction cache).
    __device__ void s3_merge_loop(unsigned long long op, unsigned long long seq, unsigned long long nodes) {
        Sv3Shared& s3 = sh->s3;
        const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
        const uint32_t mw = warp - 2u, grp = mw >> 2, gw = mw & 3u;
        const bool ml = threadIdx.x == kS3MergeLeader;
        unsigned long long t = sh->root_tk;
        unsigned long long off = rv.ops[op].offset;
        // node map: 5 bits per node 1..7 (buffer index)
        unsigned long long nbp = 0;
        for (uint32_t i = 1; i <= 7; ++i) nbp |= (unsigned long long)(i - 1) << (5 * i);
        auto nbg = [&](uint32_t i) { return (uint32_t)(nbp >> (5 * i)) & 31u; };
        auto nbs = [&](uint32_t i, uint32_t b) {
            nbp = (nbp & ~(31ull << (5 * i))) | ((unsigned long long)b << (5 * i));
        };
        uint32_t rfb = 7;                           // this op's refill buffer
        uint32_t resv = 0;                          // reserved for the control warp (previous op)
        bool req_next = false;                      // refill of op j+1 requested
        for (uint32_t j = 0;; ++j) {
            const unsigned long long t_op = now();
            // ---- buffer plan: the control warp must be done with op j-2
            if (j >= 2)
                while (s3.w0_done < j - 1) __nanosleep(20);
            uint32_t used = resv | (1u << rfb);
            for (uint32_t i = 1; i <= 7; ++i) used |= 1u << nbg(i);
            const uint32_t fr = ~used & 0xFFFFFFu;
            // the k-th free buffer: lane L holds buffer L's rank among the free ones
            const uint32_t myrank = __popc(fr & ((1u << lane) - 1u));
            const bool myfree = lane < 24 && ((fr >> lane) & 1u);
            auto scratch = [&](uint32_t k) {
                return (uint32_t)__ffs(__ballot_sync(0xFFFFFFFFu, myfree && myrank == k)) - 1u;
            };
            const uint32_t bH0 = scratch(0), blo0 = scratch(1), bH1 = scratch(2), blo1 = scratch(3),
                           bL3 = scratch(4), bR3 = scratch(5), bH2 = scratch(6), bnr = scratch(7), bc1 = scratch(8),
                           bnh1 = scratch(9), bc2 = scratch(10), bnh2 = scratch(11), brfn = scratch(12);
            // ---- the path through levels 0-1 (children batches only)
            bool mc0, el0, hl0, mc1, el1, hl1;
            const uint32_t nb2 = nbg(2), nb3 = nbg(3);
            const Key* n2 = buf(nb2);
            const Key* n3 = buf(nb3);
            s3_children(n2, n3, mc0, el0, hl0);
            const uint32_t hi1 = hl0 ? 2u : 3u, lo1 = hi1 ^ 1u;
            const Key* k1l = buf(nbg(2 * hi1));
            const Key* k1r = buf(nbg(2 * hi1 + 1));
            s3_children(k1l, k1r, mc1, el1, hl1);
            const uint32_t hi2 = hl1 ? 2u * hi1 : 2u * hi1 + 1u, lo2 = hi2 ^ 1u;
            if (ml) {
                tl(j, 0);
                // the claim warp: hi2's children
                s3.g3_t = t;
                s3.g3_op = op;
                s3.g3_j = j;
                s3.g3_hi2 = hi2;
                s3.g3_L = bL3;
                s3.g3_R = bR3;
                mb_arrive(&s3.mb_go3);
                if (j == 0) s3_go(0, nodes, rfb, op);  // the first refill is not ahead
                req_next = false;
                if (nodes - 1 >= kServeMin && s3_have(t + 1)) {
                    s3_go(j + 1, nodes - 1, brfn, s3.la_op[(t + 1) & 7u]);
                    req_next = true;
                }
            }
            // ---- level-0/1 bounds: the largest key of H0' and H1' (the k
            // smallest of the children), without merging
            const Key h0max = mc0 ? warp_kth_max<Key, K>(n2, n3) : (hl0 ? n2 : n3)[K - 1];
            const Key h1max = mc1 ? warp_kth_max<Key, K>(k1l, k1r) : (hl1 ? k1l : k1r)[K - 1];
            mb_wait(&s3.mb_rf[j & 1u], (j >> 1) & 1u);
            if (ml) tl(j, 2);
            const Key* RF = buf(rfb);
            const Key rmin = RF[0], rmax = RF[K - 1];
            const bool stop0 = rmax <= n2[0] && rmax <= n3[0];
            const bool mcur0 = !stop0 && !(elide && h0max <= rmin);  // H0'.min < refill.max: H0' <= refill is the test
            const bool stop1 = !stop0 && !mcur0 && rmax <= k1l[0] && rmax <= k1r[0];
            const bool mcur1f = !stop0 && !mcur0 && !stop1 && !(elide && h1max <= rmin);
            const bool fast = !stop0 && !mcur0 && !stop1 && !mcur1f;
            // decisions filled in below
            bool stop1g = stop1, mcur1 = false, stop2 = false, early2 = false, go2 = false, mcur2 = false;
            bool mc2 = false, el2 = false, hl2 = false;
            uint32_t lk3 = 0, rk3 = 0, lrel3 = kAvail, rrel3 = kAvail;
            uint32_t c1b = rfb, c2b = rfb;
            const uint32_t bH0p = mc0 ? bH0 : nbg(hi1);
            const uint32_t bH1p = mc1 ? bH1 : nbg(hi2);
            uint32_t bH2p = 0;
            bool c3_mbox = false;
            const uint32_t nrounds_max = fast ? 3u : 4u;
#pragma unroll 1
            for (uint32_t r = 0; r < nrounds_max; ++r) {
                const Key* A = nullptr;
                const Key* B = nullptr;
                Key* out = nullptr;
                bool second = false, global = false, act = false, copy = false;
                if (r == 0) {  // H0 || lo0 || H1 (both paths)
                    if (grp == 0) { act = mc0; A = n2; B = n3; out = buf(bH0); }
                    else if (grp == 1) { act = mc0; A = n2; B = n3; out = buf(blo0); second = true; }
                    else { act = mc1; A = k1l; B = k1r; out = buf(bH1); }
                } else if (fast || r >= 2) {
                    // level 2 decisions need the level-3 children (and, on the
                    // general path, carried 2 from round 2)
                    if ((fast && r == 1) || (!fast && r == 2)) {
                        mb_wait(&s3.mb_c3, j & 1u);
                        if (ml) tl(j, 4);
                        lk3 = s3.lk3;
                        rk3 = s3.rk3;
                        lrel3 = s3.lrel3;
                        rrel3 = s3.rrel3;
                        const Key* L3 = buf(bL3);
                        const Key* R3 = buf(bR3);
                        const bool le3 = !lk3 || L3[0] == kMaxKey, re3 = !rk3 || R3[0] == kMaxKey;
                        if (!le3 && !re3) s3_children(L3, R3, mc2, el2, hl2);
                        else hl2 = !le3;
                    }
                    const Key* L3 = buf(bL3);
                    const Key* R3 = buf(bR3);
                    if (fast && r == 1) {  // lo1 || H2 || lo2 -> HBM; level 2 with the refill
                        const bool le3 = !lk3 || L3[0] == kMaxKey, re3 = !rk3 || R3[0] == kMaxKey;
                        stop2 = le3 && re3;
                        if (!stop2 && rmax <= (le3 ? kMaxKey : L3[0]) && rmax <= (re3 ? kMaxKey : R3[0])) {
                            early2 = true;
                            stop2 = true;
                        }
                        go2 = !stop2;
                        c2b = rfb;
                        bH2p = mc2 ? bH2 : (hl2 ? bL3 : bR3);
                        // H2' (the k smallest of the level-3 children) bounds the
                        // refill's last step without merging first
                        const Key h2max = mc2 ? warp_kth_max<Key, K>(L3, R3) : buf(bH2p)[K - 1];
                        mcur2 = go2 && !(elide && h2max <= rmin);
                        if (grp == 0) { act = mc1; A = k1l; B = k1r; out = buf(blo1); second = true; }
                        else if (grp == 1) { act = go2 && mc2; A = L3; B = R3; out = buf(bH2); }
                        else {
                            act = go2 && mc2; A = L3; B = R3; second = true; global = true;
                            out = node(hl2 ? 2ull * hi2 + 1 : 2ull * hi2);
                        }
                    } else if (fast && r == 2) {  // only if the refill interleaves H2'
                        c3_mbox = true;
                        if (grp == 0) { act = true; A = RF; B = buf(bH2p); out = buf(bnh2); }
                        else if (grp == 1) { act = true; A = RF; B = buf(bH2p); out = mbox(t + 1); second = true; global = true; }
                    } else if (r == 2) {  // general: level 1 with carried 1 || H2
                        const Key* C1 = buf(c1b);
                        stop1g = !stop0 && C1[K - 1] <= k1l[0] && C1[K - 1] <= k1r[0];
                        const bool go1 = !stop0 && !stop1g;
                        mcur1 = go1 && !(elide && !needs_merge_full<Key, K>(C1, buf(bH1p)));
                        c2b = mcur1 ? bc2 : c1b;
                        if (grp == 2) { act = go1 && mc2; A = L3; B = R3; out = buf(bH2); }
                        else { act = mcur1; A = C1; B = buf(bH1p); out = buf(grp == 0 ? bnh1 : bc2); second = grp == 1; }
                    } else {  // general r == 3: level 2 with carried 2 || lo2 -> HBM
                        const bool go1 = !stop0 && !stop1g;
                        const bool le3 = !lk3 || L3[0] == kMaxKey, re3 = !rk3 || R3[0] == kMaxKey;
                        const Key* C2 = buf(c2b);
                        if (go1) {
                            stop2 = le3 && re3;
                            if (!stop2 && C2[K - 1] <= (le3 ? kMaxKey : L3[0]) && C2[K - 1] <= (re3 ? kMaxKey : R3[0])) {
                                early2 = true;
                                stop2 = true;
                            }
                        }
                        go2 = go1 && !stop2;
                        bH2p = mc2 ? bH2 : (hl2 ? bL3 : bR3);
                        mcur2 = go2 && !(elide && !needs_merge_full<Key, K>(C2, buf(bH2p)));
                        c3_mbox = mcur2;
                        if (grp == 0) { act = mcur2; A = C2; B = buf(bH2p); out = buf(bnh2); }
                        else if (grp == 1) { act = mcur2; A = C2; B = buf(bH2p); out = mbox(t + 1); second = true; global = true; }
                        else {
                            act = go2 && mc2; A = L3; B = R3; second = true; global = true;
                            out = node(hl2 ? 2ull * hi2 + 1 : 2ull * hi2);
                        }
                    }
                } else {  // general r == 1: level 0 with the refill || lo1
                    c1b = mcur0 ? bc1 : rfb;
                    if (grp == 2) { act = mc1; A = k1l; B = k1r; out = buf(blo1); second = true; }
                    else { act = mcur0; A = RF; B = buf(bH0p); out = buf(grp == 0 ? bnr : bc1); second = grp == 1; }
                }
                if (act)
                    grp_merge_half_rt<Key, K, 4>(A, B, out, gw, second, global);
                else if (copy)
                    grp_store<Key>(out, A, K, threadIdx.x & 127u, 128u);
                if (r == 0 && (threadIdx.x & 127u) == 64u) tl(j, 8u + grp);  // group leaders: merge done
                // the leader decides, before the op's last barrier, whether
                // the hold goes on (every merge thread reads it after)
                const bool last_round = fast ? (r == 2 || (r == 1 && !mcur2)) : r == 3;
                if (ml && last_round) {
                    const bool on = nodes - 1 >= kServeMin && s3_have(t + 1);
                    s3.hold_on[j & 1u] = on;
                    if (on) {
                        s3.nx_op[j & 1u] = s3.la_op[(t + 1) & 7u];
                        s3.nx_off[j & 1u] = s3.la_off[(t + 1) & 7u];
                        if (!req_next) {
                            s3_go(j + 1, nodes - 1, brfn, s3.la_op[(t + 1) & 7u]);
                            req_next = true;
                        }
                    }
                }
                grp_sync(kS3BarMerge, kS3MergeThreads);
                if (ml) tl(j, r == 0 ? 1 : r == 1 ? 3 : r == 2 ? 5 : 6);
                if (last_round) break;
            }
            // ---- the op's node map, record and counters
            const uint32_t rootb = nbg(1);
            uint32_t c3buf = 0xFFFFFFFFu;
            unsigned long long cont = 0;
            uint32_t crel = kAvail;
            const uint32_t nrb = stop0 ? rfb : (mcur0 ? bnr : bH0p);
            const uint32_t nh1b = mcur1 ? bnh1 : bH1p;
            const bool go1 = !stop0 && !(fast ? stop1 : stop1g);
            nbs(1, nrb);
            if (!stop0) {
                if (mc0) nbs(lo1, blo0);
                nbs(hi1, go1 ? (fast ? bH1p : nh1b) : c1b);
                if (go1) {
                    if (mc1) nbs(lo2, blo1);
                    nbs(hi2, stop2 ? c2b : (mcur2 ? bnh2 : bH2p));
                }
            }
            const unsigned long long hi3 = hl2 ? 2ull * hi2 : 2ull * hi2 + 1, lo3 = hi3 ^ 1ull;
            if (go2) {
                cont = hi3;
                crel = hl2 ? lrel3 : rrel3;
                if (!c3_mbox) c3buf = c2b;  // the carried batch moves down unchanged
            }
            const bool on = s3.hold_on[j & 1u] != 0;
            if (ml) {
                Sv3Rec& R = s3.rec[j & 3u];
                uint32_t merges = 0, elided = 0, early = 0, visits = 0;
                if (stop0) {
                    ++early;
                } else {
                    merges += mc0 + mcur0;
                    elided += el0 + !mcur0;
                    ++visits;
                    if (!go1) {
                        ++early;
                    } else {
                        merges += mc1 + mcur1;
                        elided += el1 + !mcur1;
                        ++visits;
                        if (stop2) {
                            early += early2;
                        } else {
                            merges += mc2 + mcur2;
                            elided += el2 + !mcur2;
                            ++visits;
                        }
                    }
                }
                R.op = op;
                R.off = off;
                R.seq = seq;
                R.t = t;
                R.cont = cont;
                R.crel = crel;
                R.rootbuf = rootb;
                R.c3buf = c3buf;
                R.cnt_merges = merges;
                R.cnt_elided = elided;
                R.cnt_early = early;
                R.cnt_visits = visits;
                R.last = !on;
                uint32_t nrel = 0;
                if (go2) {
                    if (hl2 ? rk3 : lk3) {
                        R.relslot[0] = lo3;
                        R.relst[0] = hl2 ? rrel3 : lrel3;
                        nrel = 1;
                    }
                } else {
                    if (lk3) {
                        R.relslot[nrel] = 2ull * hi2;
                        R.relst[nrel++] = lrel3;
                    }
                    if (rk3) {
                        R.relslot[nrel] = 2ull * hi2 + 1;
                        R.relst[nrel++] = rrel3;
                    }
                }
                R.nrel = nrel;
                // the words the control warp's releases will produce: the next
                // claims of these nodes CAS them directly
                for (uint32_t i = 0; i < nrel; ++i) {
                    const uint32_t x = (uint32_t)R.relslot[i] - 8u;
                    s3.w3pred[x] = s3.w3in[x] + 8u + R.relst[i] - kInUse;
                }
                if (cont) s3.w3pred[(uint32_t)cont - 8u] = 0xFFFFFFFFu;
                if (record) {  // the op's turn at nodes 1-7 ends; the next op's begins
                    for (unsigned long long i = 1; i <= 7; ++i) rec_for(op, kEvRel, i);
                    if (on)
                        for (unsigned long long i = 1; i <= 7; ++i) rec_for(s3.nx_op[j & 1u], kEvAcq, i);
                }
                if (prof) {
                    atomicAdd(&hv.prof[pf3Ops], 1ull);
                    atomicAdd(&hv.prof[pf3Op], now() - t_op);
                    atomicAdd(&hv.prof[fast ? pf3R0 : pf3R1], 1ull);
                }
                // one record phase at a time: the control warp has taken the last one
                while (s3.w0_seen < j) __nanosleep(20);
                mb_arrive(&s3.mb_rec);
            }
            resv = (1u << rootb) | (c3buf != 0xFFFFFFFFu ? 1u << c3buf : 0u);
            rfb = brfn;
            if (!on) {
                if (ml) {  // the refill and claim warps leave; hold-end state
                    s3_go(j + 1, 0, 0, 0);
                    s3_go(j + 2, 0, 0, 0);
                    s3.g3_hi2 = 0;
                    mb_arrive(&s3.mb_go3);
                    for (uint32_t i = 1; i <= 7; ++i) s3.nb_end[i] = nbg(i);
                    sh->nodes = nodes - 1;
                }
                break;
            }
            ++t;
            op = s3.nx_op[j & 1u];
            off = s3.nx_off[j & 1u];
            ++seq;
            --nodes;
        }
    }

    // Merge leader: a refill request for op j (rank 0 = leave the loop).
    __device__ void s3_go(uint32_t j, unsigned long long rank, uint32_t b, unsigned long long op) {
        Sv3Shared& s3 = sh->s3;
        s3.go_last[j & 1u] = rank;
        s3.go_j[j & 1u] = j;
        s3.go_buf[j & 1u] = b;
        s3.go_op[j & 1u] = op;
        mb_arrive(&s3.mb_go[j & 1u]);
    }

    __device__ void do_delete(unsigned long long opi, const bh_op& o) {
        const unsigned long long t0 = now();
        rec(kEvInv, 0);
        if (leader()) {
            uint32_t gated = 0;
            if (hv.variant == BH_BU) {
                // BU phase gate: a delete that will heapify (>= 2 nodes) waits
                // until no bottom-up climb is in flight.  The request lets a
                // delete server ahead in the queue run this op (serve_deletes).
                const bool can_post = T >= 128 && (hv.flags & kDbgNoDelServe) == 0;
                for (;;) {
                    if (root_lock(false, false, can_post)) {
                        gated = 2;  // served: counted in the gate by the server
                        break;
                    }
                    const unsigned long long nodes_now = ld_cg_u64(&hdr->node_count);
                    if (nodes_now < 2) break;
                    if (gate_try(false)) {
                        gated = 1;
                        break;
                    }
                    root_unlock(false);
                    gate_wait(false);
                }
                if (gated != 2) rec(kEvAcq, 1);
            } else {
                // TD: no phase gate; the request lets a delete server run it
                const bool can_post = T >= 128 && (hv.flags & kDbgNoDelServe) == 0;
                if (root_lock(true, false, can_post)) gated = 2;
            }
            sh->owned = gated;
        }
        const unsigned long long t1 = now();
        __syncthreads();
        if (sh->owned == 2) {
            // a delete server ran this op's top levels and wrote its result;
            // this CTA runs the continuation of the op served before it
            const unsigned long long tk = sh->root_tk;
            const unsigned long long cont = sh->contw & 0x7FFFFFFFu;
            const uint32_t crel = (sh->contw >> 31) ? kDelMod : kAvail;
            if (record) {  // its lock events and response are that op's
                if (leader()) sh->op_next = ld_cg_u64(reinterpret_cast<const unsigned long long*>(qline(tk) + 14));
                __syncthreads();
                cur_op = sh->op_next;
            }
            if (cont) {
                // the carried batch travels while the node's children are claimed
                cta_load_async<Key, T>(buf(0), mbox(tk), K);
                acquire_children(cont, buf(1), buf(2));
                cp_async_wait_all();
                __syncthreads();
                heapify_down(0, t1, true, cont, crel);
            }
            rec(kEvRes, 0);
            if (hv.variant == BH_BU && leader()) gate_leave(false);
            return;
        }
        const bool gated = sh->owned != 0;
        // the root batch, read in the same round trip as the header
        Key* cur_s = buf(0);
        if (leader()) {
            sh->nodes = ld_cg_u64(&hdr->node_count);
            sh->plen = ld_cg_u64(&hdr->partial_len);
            sh->seq = ld_cg_u64(&hdr->delete_count);
            // peek (relaxed, same round trip) at the next ticket's serve
            // request; TD heaps start serving only for a run of deletes (two
            // queued), short runs between inserts do not pay for it
            const unsigned long long t1q = sh->root_tk + 1;
            bool peek = __ldcg(qline(t1q) + 11) == ((((uint32_t)t1q) << 1) | 1u);
            if (hv.variant == BH_TD)
                peek = peek && __ldcg(qline(t1q + 1) + 11) == ((((uint32_t)t1q + 1u) << 1) | 1u);
            sh->serve = peek;
        }
        cta_load<Key, T>(cur_s, node(1), K);
        __syncthreads();
        const unsigned long long nodes = sh->nodes;
        const uint32_t plen = (uint32_t)sh->plen;
        const unsigned long long seq = sh->seq;
        Key* out = static_cast<Key*>(rv.out_pool) + o.offset;
        // warm L2 with the refill nodes of the next few deletes (HBM-cold
        // bottom-level nodes; the claim then hits L2)
        if (threadIdx.x >= 32 && threadIdx.x < 32 + kRefillAhead && nodes > threadIdx.x - 32 + 5) {
            const unsigned long long slot = slot_for_rank(nodes - 1 - (threadIdx.x - 32));
            const char* a = reinterpret_cast<const char*>(node(slot));
            for (uint32_t off = 0; off < kNodeBytes; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a + off));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(st(slot)));
        }
        pf_add(pfDelOps, 1);
        pf_add(pfDelRootWait, t1 - t0);

        if (nodes == 0) {
            if (plen == 0) {  // empty heap (heap.cpp:424-429)
                if (leader()) lane_unlock(1);
                pf_add(pfDelRootHold, now() - t1);
                status(opi, BH_E_EMPTY, 0, ~0ull);
                rec(kEvRes, 0);
                return;
            }
            // fewer than k keys: they all live in the partial buffer
            cta_copy_gg<Key, T>(out, partial, plen);
            count(cDeletes);
            __syncthreads();
            if (leader()) {
                st_cg_u64(&hdr->partial_len, 0);
                st_cg_u64(&hdr->delete_count, seq + 1);
                lane_unlock(1);
            }
            pf_add(pfDelRootHold, now() - t1);
            status(opi, BH_OK, plen, seq);
            rec(kEvRes, 0);
            return;
        }

        // delete serving: with waiting deletes queued behind, this CTA keeps
        // the root and runs their top levels too
        if (T >= 128 && (gated || hv.variant == BH_TD) && plen == 0 && nodes >= kServeMin &&
            (hv.flags & kDbgNoDelServe) == 0) {
            if (leader() && sh->serve) {
                unsigned long long nop = 0;
                sh->serve = waiting_delete(sh->root_tk + 1, nop);
            }
            __syncthreads();
            if (sh->serve) {
                if constexpr (kS3) {
                    if (hv.flags & kDbgServe3) {
                        serve3(opi, seq, nodes);
                        return;
                    }
                }
                serve_deletes(opi, seq, nodes);
                return;
            }
        }
        cta_store<Key, T>(out, cur_s, K);  // the result: the root's k keys
        if (leader()) {
            if (cur_s[K - 1] == kMaxKey)
                atomicOr(&hdr->error_flags, (unsigned long long)kErrSentinelEscaped);
            st_cg_u64(&hdr->delete_count, seq + 1);
            st_cg_u64(&hdr->node_count, nodes - 1);
        }
        count(cDeletes);
        if (nodes == 1) {
            cta_fill<Key, T>(node(1), kMaxKey, K);
            __syncthreads();
            if (leader()) lane_unlock(1);
            pf_add(pfDelRootHold, now() - t1);
            status(opi, BH_OK, K, seq);
            rec(kEvRes, 0);
            if (gated && leader()) gate_leave(false);
            return;
        }

        // ---- refill_root_from(last) (heap.cpp:467-531): only the root is
        // held while the last node is claimed.  With nodes >= 4 the last node
        // is below level 1, so one half of the CTA claims, copies, blanks and
        // releases it while the other half claims the root's children (the
        // first heapify level) -- the refill never waits on a child, so the
        // reference's deadlock argument (last released before any child is
        // awaited) still holds for the refill half, and the children half
        // holds nothing but the root while it waits ----
        const unsigned long long last = slot_for_rank(nodes);
        Key* sp = buf(3);
        const unsigned long long ta = now();
        pf_add(pfRsHead, ta - t1);
        if (plen) cta_load<Key, T>(sp, partial, plen);
        // (recorded heaps run the same schedule; their histories mark the
        // refill span, which may overlap the children's claims)
        const bool split = T >= 64 && nodes >= 4;
        if (split) {
            constexpr uint32_t kHalf = T / 2;
            if (threadIdx.x < kHalf) {
                refill_last(last, cur_s, 0, kHalf, 1);
                pf_add(pfSplitA, now() - ta);
            } else {
                acquire_children(1, buf(1), buf(2), kHalf, kHalf, 2);
                if (prof && threadIdx.x == kHalf) atomicAdd(&hv.prof[pfSplitB], now() - ta);
            }
            __syncthreads();
        } else {
            refill_last(last, cur_s, 0, T, 0);
        }
        const unsigned long long td = now();
        pf_add(pfRsLast, td - ta);

        // ---- remerge_root_with_partial (heap.cpp:533-545) ----
        int ci = 0;
        if (plen) {
            if (elide && sp[0] >= cur_s[K - 1]) {
                count(cElided);
            } else {
                Key* tmp = buf(5);
                cta_merge<Key, T>(cur_s, K, sp, plen, tmp, K, partial);
                count(cMerges);
                note_partial(plen);
                ci = 5;
            }
            __syncthreads();
        }
        pf_add(pfRsFill, now() - td);
        heapify_down(ci, t1, split);
        if (gated && leader()) gate_leave(false);
        status(opi, BH_OK, K, seq);
        rec(kEvRes, 0);
    }

    // heapify_down (heap.cpp:591-667) with the carried batch in buf(ci).
    // Root held on entry.  Releases every lock it holds.
    //
    // Per level (acquire_child, early stop, hi/lo with the tie fix, then the
    // two merges of heap.cpp:637-660), scheduled for a short critical path:
    //   phase 1  the node's new batch = first half of merge(cur, H), where H
    //            is the first half of merge(L, R) (the k smallest of the
    //            children); written, and the node released at once;
    //   phase 2  threads [0, T/2) compute the carried batch (second half of
    //            merge(cur, H)) and the lo child's batch (second half of
    //            merge(L, R)) and release the lo child; threads [T/2, T)
    //            meanwhile claim and load hi's children and, when they
    //            interleave, already compute the next level's H.
    // A node is held only for phase 1 of its own level; the next level's
    // claim round trip and H merge run in the shadow of the second halves.
    // Lock order, states and released contents are the reference's.
    // `pre`: the root's children are already claimed, in buf(1) and buf(2).
    // `start`/`start_rel`: a served delete's continuation starts below the
    // levels its server ran, at a node the server claimed (serve_one).
    __device__ void heapify_down(int ci, unsigned long long t_root, bool pre, unsigned long long start = 1,
                                 uint32_t start_rel = kAvail) {
        constexpr bool kSplit = T >= 64;
        constexpr uint32_t kHalf = kSplit ? T / 2 : T;
        // upper-half lane with no claim duty (acquire_children polls with its
        // first two lanes)
        constexpr uint32_t kRelLane = kSplit ? (T >= 128 ? kHalf + 32 : kHalf + 2) : 0;
        unsigned long long cur = start;
        uint32_t cur_rel = start_rel;
        const unsigned long long t_start = now();
        auto free_buf = [](uint32_t used) { return __ffs(~used) - 1; };
        int li, ri;
        if (pre) {
            li = 1;
            ri = 2;
        } else {
            li = free_buf(1u << ci);
            ri = free_buf((1u << ci) | (1u << li));
        }
        bool have = pre;  // children of cur claimed and loaded
        int hx = -1;      // buffer holding H, when precomputed
        for (;;) {
            Key* cur_s = buf(ci);
            const unsigned long long l = 2 * cur, r = 2 * cur + 1;
            const unsigned long long tl0 = now();
            if (!have) acquire_children(cur, buf(li), buf(ri));
            if (cur == 1) pf_add(pfRsChild, now() - tl0);
            else pf_add(pfLvAcq, now() - tl0);
            const unsigned long long tl2 = now();
            pf_add(pfLevels, 1);
            Key* L = buf(li);
            Key* R = buf(ri);
            const uint32_t lk = sh->lk, rk = sh->rk;
            const uint32_t lrel = sh->lrel, rrel = sh->rrel;
            const bool lempty = !lk || L[0] == kMaxKey;
            const bool rempty = !rk || R[0] == kMaxKey;
            const Key cmax = cur_s[K - 1];
            bool stop = lempty && rempty;
            if (!stop) {
                const Key lmin = lempty ? kMaxKey : L[0];
                const Key rmin = rempty ? kMaxKey : R[0];
                if (cmax <= lmin && cmax <= rmin) {
                    count(cEarlyStops);
                    stop = true;
                }
            }
            if (stop) {
                cta_store<Key, T>(node(cur), cur_s, K);
                __syncthreads();
                if (leader()) {
                    if (lk) lane_unlock(l, lrel);
                    if (rk) lane_unlock(r, rrel);
                    lane_unlock(cur, cur_rel);
                }
                if (cur == 1) pf_add(pfDelRootHold, now() - t_root);
                pf_add(pfDelRest, now() - t_start);
                return;
            }
            // Merge the children: lo lands in the child whose max was larger
            // (right on ties), hi in the other, which we descend into.
            bool hi_left;
            bool merge_children = false;
            if (lempty) {
                hi_left = false;
            } else if (rempty) {
                hi_left = true;
            } else if (elide && !needs_merge_full<Key, K>(L, R)) {
                count(cElided);
                // fix of heap.cpp:628-636: the batch with the smaller keys is hi
                hi_left = L[K - 1] <= R[0];
            } else {
                hi_left = !(L[K - 1] > R[K - 1]);
                merge_children = true;
                count(cMerges);
            }
            const unsigned long long hi = hi_left ? l : r;
            const unsigned long long lo = hi_left ? r : l;
            const uint32_t lo_locked = hi_left ? rk : lk;
            const uint32_t hi_rel = hi_left ? lrel : rrel;
            const uint32_t lo_rel = hi_left ? rrel : lrel;
            prefetch_node(2 * hi);  // warm L2 with the next level
            prefetch_node(2 * hi + 1);
            // ---- phase 1 ----
            if (merge_children && hx < 0) {  // H not precomputed (root level)
                hx = free_buf((1u << ci) | (1u << li) | (1u << ri));
                grp_merge_half<Key, K, T / 32, false, false>(L, R, buf(hx), threadIdx.x >> 5);
                // every thread reads H's ends below (merge_cur decides the
                // buffer plan), so the whole CTA waits for it
                __syncthreads();
            }
            Key* hdata = merge_children ? buf(hx) : (hi_left ? L : R);
            const bool merge_cur = !(elide && !needs_merge_full<Key, K>(cur_s, hdata));
            if (merge_cur) count(cMerges);
            else count(cElided);
            count(cVisits);
            if (!merge_cur)  // early stop ruled out the ordered case: a full inversion
                cta_store<Key, T>(node(cur), hdata, K);
            else
                grp_merge_half<Key, K, T / 32, false, true>(cur_s, hdata, node(cur), threadIdx.x >> 5);
            const unsigned long long tl3 = now();
            __syncthreads();
            // The release fence waits for the batch's stores to be acked; a
            // thread of the upper half (idle until its claim) pays it, so the
            // lower half starts the carried-batch merge at once.
            if (threadIdx.x == kRelLane) {
                lane_unlock(cur, cur_rel);
                if (lo_locked && !merge_children) lane_unlock(lo, lo_rel);  // unchanged
            }
            if (cur == 1) pf_add(pfDelRootHold, now() - t_root);
            // ---- phase 2 ----
            uint32_t used = (1u << ci) | (1u << li) | (1u << ri) | (merge_children ? (1u << hx) : 0u);
            const int nxi = merge_cur ? free_buf(used) : ci;
            used |= 1u << nxi;
            const int li2 = free_buf(used);
            used |= 1u << li2;
            const int ri2 = free_buf(used);
            used |= 1u << ri2;
            const int hx2 = free_buf(used);
            bool h2 = false;
            if constexpr (kSplit) {
                if (threadIdx.x < kHalf) {
                    // the carried batch and the lo child's batch side by side
                    // on two quarter groups (one after the other below 128
                    // threads)
                    constexpr int kQW = kHalf / 64;
                    const uint32_t w = threadIdx.x >> 5;
                    if constexpr (kQW >= 1) {
                        if (w < (uint32_t)kQW) {
                            if (merge_cur) grp_merge_half<Key, K, kQW, true, false>(cur_s, hdata, buf(nxi), w);
                        } else if (merge_children) {
                            grp_merge_half<Key, K, kQW, true, true>(L, R, node(lo), w - kQW);
                        }
                    } else {
                        if (merge_cur) grp_merge_half<Key, K, 1, true, false>(cur_s, hdata, buf(nxi), 0);
                        if (merge_children) grp_merge_half<Key, K, 1, true, true>(L, R, node(lo), 0);
                    }
                    grp_sync(1, kHalf);
                    if (merge_children && leader() && lo_locked) lane_unlock(lo, lo_rel);
                } else {
                    acquire_children(hi, buf(li2), buf(ri2), kHalf, kHalf, 2);
                    // the next level's H, if its children interleave (the same
                    // test the next level makes)
                    const Key* L2 = buf(li2);
                    const Key* R2 = buf(ri2);
                    const bool e2 = !sh->lk || L2[0] == kMaxKey || !sh->rk || R2[0] == kMaxKey;
                    if (!e2 && !(elide && !needs_merge_full<Key, K>(L2, R2)))
                        grp_merge_half<Key, K, kHalf / 32, false, false>(L2, R2, buf(hx2), (threadIdx.x - kHalf) >> 5);
                }
                __syncthreads();
                const Key* L2 = buf(li2);
                const Key* R2 = buf(ri2);
                const bool e2 = !sh->lk || L2[0] == kMaxKey || !sh->rk || R2[0] == kMaxKey;
                h2 = !e2 && !(elide && !needs_merge_full<Key, K>(L2, R2));
                have = true;
                li = li2;
                ri = ri2;
            } else {
                if (merge_cur) grp_merge_half<Key, K, T / 32, true, false>(cur_s, hdata, buf(nxi), threadIdx.x >> 5);
                if (merge_children) grp_merge_half<Key, K, T / 32, true, true>(L, R, node(lo), threadIdx.x >> 5);
                __syncthreads();
                if (leader() && lo_locked && merge_children) lane_unlock(lo, lo_rel);
                have = false;
                li = free_buf(1u << nxi);
                ri = free_buf((1u << nxi) | (1u << li));
            }
            pf_add(pfLvMerge, tl3 - tl2);
            pf_add(pfLvRel, now() - tl3);
            hx = h2 ? hx2 : -1;
            cur = hi;
            cur_rel = hi_rel;
            ci = nxi;
        }
    }
};

template <typename Key, int K, int T, bool Rec>
__global__ void __launch_bounds__(T, (512 / T > 0 ? 512 / T : 1)) heap_ops_kernel(HeapView hv, RunView rv) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ OpShared sh;
    HeapCta<Key, K, T, Rec> cta(hv, rv, smem_raw, &sh);
    cta.run();
}

#ifndef BH_THREADS_CAP
#define BH_THREADS_CAP 512
#endif
#ifndef BH_THREADS_DIV
#define BH_THREADS_DIV 2
#endif
// One CTA per op: K/2 threads (two merge outputs per thread per 2K-merge),
// capped; both knobs are build-time for tuning sweeps.
template <typename Key, int K>
struct KernelCfg {
    static constexpr int kWant = K / BH_THREADS_DIV;
    static constexpr int kThreads = kWant < 32 ? 32 : (kWant > BH_THREADS_CAP ? BH_THREADS_CAP : kWant);
    // 10 node buffers, 24 where the three-level delete server runs; + window over-read pad
    static constexpr uint32_t kSmem = (Serve3Cfg<Key, K, kThreads>::kOn ? 24u : 10u) * K * sizeof(Key) + 64;
};

}  // namespace bh

// mb_handoff.cu -- latency of handing a 4 KiB node (K=1024 u32 keys) from
// one CTA to another on a different SM (tooling).  Two CTAs of 512 threads
// ping-pong the node; SM cycles per one-way hand-off, as seen by CTA 0.
//
// The heap's continuation hand-off today is mode 0: the node staged in an
// HBM mailbox by st.global.cg, a CTA barrier, a GPU-scope fence and a flag;
// the woken CTA acquires the flag and loads the node.  The other modes are the
// Blackwell alternatives DESIGN.md section 6 asks about:
//   1  HBM mailbox + flag, receiver pulls the node with a TMA bulk copy
//      (cp.async.bulk global -> shared, mbarrier complete_tx)
//   2  TMA bulk store (shared -> global) + wait_group + fence + flag, receiver
//      as mode 0
//   3  flag only (no data), GPU scope: the signal floor through L2
//   4  DSMEM: st.shared::cluster of the node into the peer CTA's buffer, CTA
//      barrier, remote mbarrier arrive (release.cluster), acquire.cluster wait
//   5  DSMEM bulk copy (cp.async.bulk shared::cta -> shared::cluster) with
//      complete_tx on the peer's mbarrier
//   6  remote mbarrier arrive only (no data): the cluster signal floor
// Modes 0-3 are run without and with a 2-CTA cluster (placement only), 4-6
// need the cluster.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long clk() {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
    return c;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void wait_parity(uint32_t mb, uint32_t par, bool cluster_acq) {
    uint32_t ok = 0;
    while (!ok) {
        if (cluster_acq)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(mb), "r"(par) : "memory");
        else
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(mb), "r"(par) : "memory");
    }
}
__device__ __forceinline__ void spin_flag(const unsigned* f, unsigned want) {
    unsigned v;
    do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    } while (v != want);
}
__device__ __forceinline__ void post_flag(unsigned* f, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

struct Args {
    int mode, iters, clustered;
    uint4* mbox;                // 2 x 4 KiB
    unsigned* flags;            // 2 words, 128 B apart
    unsigned long long* out;    // [cycles/one-way, smid0, smid1, checksum]
};

__global__ void __launch_bounds__(512, 1) handoff(Args a) {
    __shared__ __align__(128) uint4 buf[256];
    __shared__ __align__(8) unsigned long long mb;
    const uint32_t tid = threadIdx.x, me = blockIdx.x, peer = me ^ 1;
    if (tid < 256) buf[tid] = make_uint4(tid, me, 0, 0);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        uint32_t s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        a.out[1 + me] = s;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (a.clustered) cg::this_cluster().sync();
    const uint32_t mb_l = su32(&mb);
    const uint32_t mb_r = a.clustered ? mapa(mb_l, peer) : 0;
    const uint32_t buf_r = a.clustered ? mapa(su32(buf), peer) : 0;
    uint4* rbuf = a.clustered ? cg::this_cluster().map_shared_rank(buf, peer) : nullptr;
    uint32_t got = 0;  // hand-offs received (mbarrier phases)
    unsigned long long t0 = clk();
    for (int it = 0; it < a.iters; ++it) {
        const bool send = (uint32_t)(it & 1) == me;
        const unsigned seq = it + 1;
        if (send) {
            if (tid < 256) buf[tid].z += 1;  // the sender touches the node
            switch (a.mode) {
            case 0:
                if (tid < 256) __stcg(a.mbox + peer * 256 + tid, buf[tid]);
                __syncthreads();
                if (tid == 0) { __threadfence(); post_flag(a.flags + peer * 32, seq); }
                break;
            case 1:
                if (tid < 256) __stcg(a.mbox + peer * 256 + tid, buf[tid]);
                __syncthreads();
                if (tid == 0) { __threadfence(); post_flag(a.flags + peer * 32, seq); }
                break;
            case 2:
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncthreads();
                if (tid == 0) {
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;"
                                 ::"l"(a.mbox + peer * 256), "r"(su32(buf)) : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    __threadfence();
                    post_flag(a.flags + peer * 32, seq);
                }
                break;
            case 3:
                __syncthreads();
                if (tid == 0) { __threadfence(); post_flag(a.flags + peer * 32, seq); }
                break;
            case 4:
                if (tid < 256) rbuf[tid] = buf[tid];
                __syncthreads();
                if (tid == 0)
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mb_r) : "memory");
                break;
            case 5:
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncthreads();
                if (tid == 0)
                    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                                 ::"r"(buf_r), "r"(su32(buf)), "r"(mb_r) : "memory");
                break;
            case 6:
                __syncthreads();
                if (tid == 0)
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mb_r) : "memory");
                break;
            }
        } else {
            const uint32_t par = got & 1;
            ++got;
            switch (a.mode) {
            case 0:
            case 2:
                if (tid == 0) spin_flag(a.flags + me * 32, seq);
                __syncthreads();
                if (tid < 256) buf[tid] = __ldcg(a.mbox + me * 256 + tid);
                __syncthreads();
                break;
            case 1:
                if (tid == 0) {
                    spin_flag(a.flags + me * 32, seq);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(mb_l) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                                 ::"r"(su32(buf)), "l"(a.mbox + me * 256), "r"(mb_l) : "memory");
                    wait_parity(mb_l, par, false);
                }
                __syncthreads();
                break;
            case 3:
                if (tid == 0) spin_flag(a.flags + me * 32, seq);
                __syncthreads();
                break;
            case 4:
            case 6:
                if (tid == 0) wait_parity(mb_l, par, true);
                __syncthreads();
                break;
            case 5:
                if (tid == 0) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(mb_l) : "memory");
                    wait_parity(mb_l, par, false);
                }
                __syncthreads();
                break;
            }
        }
    }
    unsigned long long t1 = clk();
    if (a.clustered) cg::this_cluster().sync();  // no CTA exits while its smem may be written
    if (me == 0 && tid == 0) a.out[0] = (t1 - t0) / a.iters;
    if (me == 0 && tid < 256) atomicAdd(a.out + 3, (unsigned long long)buf[tid].z);
}


// Node loads inside one CTA (L2-resident source, as the heap's nodes are):
// n nodes of 4 KiB into shared memory, then a CTA barrier.  mode 0: ld.cg
// uint4 loop (the heap's cta_load); 1: cp.async.cg 16 B (LDGSTS) + wait_all;
// 2: one cp.async.bulk per node issued by one thread, mbarrier complete_tx.
__global__ void __launch_bounds__(512, 1) node_load(int mode, int n, int iters, const uint4* g,
                                                    unsigned long long* out) {
    __shared__ __align__(128) uint4 buf[3 * 256];
    __shared__ __align__(8) unsigned long long mb;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb)) : "memory");
    __syncthreads();
    unsigned long long acc = 0, t0 = 0;
    for (int it = -8; it < iters; ++it) {
        if (it == 0) t0 = clk();
        const uint4* src = g + (it & 7) * 3 * 256;  // 8 rotating L2-resident node triples
        if (mode == 0) {
            for (uint32_t i = tid; i < 256u * n; i += 512) buf[i] = __ldcg(src + i);
        } else if (mode == 1) {
            for (uint32_t i = tid; i < 256u * n; i += 512)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(buf + i)), "l"(src + i) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_all;" ::: "memory");
        } else {
            if (tid == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb)), "r"(4096 * n) : "memory");
                for (int j = 0; j < n; ++j)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                                 ::"r"(su32(buf + 256 * j)), "l"(src + 256 * j), "r"(su32(&mb)) : "memory");
                wait_parity(su32(&mb), (uint32_t)((it + 8) & 1), false);
            }
        }
        __syncthreads();
        acc += buf[(tid * 7) % (256 * n)].x;  // consume
        __syncthreads();
    }
    unsigned long long t1 = clk();
    if (tid == 0) out[0] = (t1 - t0) / iters;
    if (acc == 12345) out[1] = acc;
}

int main() {
    unsigned long long* o;
    uint4* mbox;
    unsigned* flags;
    CK(cudaMalloc(&o, 4 * 8));
    CK(cudaMalloc(&mbox, 2 * 4096));
    CK(cudaMalloc(&flags, 2 * 128));
    const char* names[] = {"HBM mailbox st.cg + fence + flag, ld.cg", "HBM mailbox + flag, TMA bulk load",
                           "TMA bulk store + fence + flag, ld.cg", "flag only (GPU scope)",
                           "DSMEM st + remote mbarrier arrive", "DSMEM bulk copy + complete_tx",
                           "remote mbarrier arrive only"};
    const int iters = 4000;
    for (int mode = 0; mode <= 6; ++mode) {
        for (int cl = 0; cl <= 1; ++cl) {
            if (mode >= 4 && !cl) continue;
            CK(cudaMemset(flags, 0, 2 * 128));
            CK(cudaMemset(o, 0, 4 * 8));
            Args a{mode, iters, cl, mbox, flags, o};
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            cfg.gridDim = dim3(2);
            cfg.blockDim = dim3(512);
            if (cl) {
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = 2;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
            }
            CK(cudaLaunchKernelEx(&cfg, handoff, a));
            CK(cudaDeviceSynchronize());
            unsigned long long h[4];
            CK(cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost));
            // each CTA bumps z once per send: CTA 0's final node carries iters/2 bumps
            // from each side in the data-moving modes
            const bool moves = mode != 3 && mode != 6;
            const unsigned long long want = moves ? 256ull * iters : 256ull * (iters / 2);
            printf("handoff %-42s %-9s smid %3llu -> %3llu : %5llu cycles one-way  (data %s)\n", names[mode],
                   cl ? "cluster2" : "no-cluster", h[1], h[2], h[0], h[3] == want ? "ok" : "MISMATCH");
        }
    }
    uint4* g;
    CK(cudaMalloc(&g, 8 * 3 * 4096));
    CK(cudaMemset(g, 1, 8 * 3 * 4096));
    const char* lnames[] = {"ld.cg uint4 loop", "cp.async.cg 16 B (LDGSTS)", "cp.async.bulk (TMA 1-D)"};
    for (int n = 1; n <= 3; ++n)
        for (int mode = 0; mode <= 2; ++mode) {
            node_load<<<1, 512>>>(mode, n, 2000, g, o);
            CK(cudaDeviceSynchronize());
            unsigned long long c;
            CK(cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost));
            printf("load %d x 4 KiB %-28s : %5llu cycles (incl. 2 CTA barriers)\n", n, lnames[mode], c);
        }
    return 0;
}

// bt_check.cu -- exhaustive-ish correctness check of grp_merge_half (warp-tile
// bitonic half merge, bh_select.cuh) against std::merge: both halves, K in
// {32..2048}, group sizes 1..16 warps, u32/u64, duplicates and sentinel tails.
// Tooling: make -C tools/microbench bt_check && tools/microbench/bt_check
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include "../../paper_1906_06504_b200/csrc/bh_select.cuh"
using namespace bh;
static uint32_t* replay_buf = nullptr;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

template <typename Key, int K, int NW, bool Second, bool Global = true>
__global__ void kern(const Key* in, Key* out, int rows) {
    extern __shared__ __align__(16) unsigned char sm[];
    Key* A = reinterpret_cast<Key*>(sm);
    Key* B = A + K;
    for (int r = 0; r < rows; ++r) {
        for (int i = threadIdx.x; i < 2 * K; i += blockDim.x) A[i] = in[(size_t)r * 2 * K + i];
        __syncthreads();
        if constexpr (Global) {
            grp_merge_half<Key, K, NW, Second, true>(A, B, out + (size_t)r * K, threadIdx.x >> 5);
        } else {
            Key* S = B + K;
            grp_merge_half<Key, K, NW, Second, false>(A, B, S, threadIdx.x >> 5);
            __syncthreads();
            for (int i = threadIdx.x; i < K; i += blockDim.x) out[(size_t)r * K + i] = S[i];
        }
        __syncthreads();
    }
}

template <typename Key, int K, int NW, bool Second, bool Global = true>
int run(int mode) {
    const int rows = 64;
    std::mt19937_64 rng(K * 131 + NW * 7 + Second + mode * 1000);
    std::vector<Key> h((size_t)rows * 2 * K), ref((size_t)rows * K), got((size_t)rows * K);
    const Key kMax = KeyLimits<Key>::kMax;
    for (int r = 0; r < rows; ++r) {
        Key* a = &h[(size_t)r * 2 * K];
        for (int i = 0; i < 2 * K; ++i) {
            Key v;
            if (mode == 0) v = (Key)(rng() >> 8);
            else if (mode == 1) v = (Key)(rng() % 7);             // heavy duplicates
            else v = (Key)(rng() % 1000);
            a[i] = v;
        }
        // sentinel tails / all-sentinel batches
        int ta = mode == 2 ? (int)(rng() % (K + 1)) : 0, tb = mode == 2 ? (int)(rng() % (K + 1)) : 0;
        if (mode == 2 && r % 5 == 0) ta = K;
        if (mode == 3) {  // skewed: A wide, B narrow (heap carried vs H)
            for (int i = 0; i < K; ++i) a[i] = (Key)(2134677011ull + (rng() % (4293375849ull - 2134677011ull)));
            for (int i = K; i < 2 * K; ++i) a[i] = (Key)(2163915217ull + (rng() % (2876814050ull - 2163915217ull)));
        }
        if (mode == 4 && replay_buf) { for (int i = 0; i < 2 * K; ++i) a[i] = (Key)replay_buf[i]; }
        for (int i = K - ta; i < K; ++i) a[i] = kMax;
        for (int i = 2 * K - tb; i < 2 * K; ++i) a[i] = kMax;
        std::sort(a, a + K);
        std::sort(a + K, a + 2 * K);
        std::vector<Key> m(2 * K);
        std::merge(a, a + K, a + K, a + 2 * K, m.begin());
        std::copy(m.begin() + (Second ? K : 0), m.begin() + (Second ? 2 * K : K), ref.begin() + (size_t)r * K);
    }
    Key *din, *dout;
    CK(cudaMalloc(&din, h.size() * sizeof(Key)));
    CK(cudaMalloc(&dout, got.size() * sizeof(Key)));
    CK(cudaMemcpy(din, h.data(), h.size() * sizeof(Key), cudaMemcpyHostToDevice));
    auto k = kern<Key, K, NW, Second, Global>;
    const int smem = 3 * K * sizeof(Key);
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k<<<1, 32 * NW, smem>>>(din, dout, rows);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(got.data(), dout, got.size() * sizeof(Key), cudaMemcpyDeviceToHost));
    cudaFree(din); cudaFree(dout);
    if (got != ref) {
        size_t i = 0;
        while (got[i] == ref[i]) ++i;
        printf("FAIL key=%zu K=%d NW=%d second=%d mode=%d at %zu (row %zu pos %zu): got %llu want %llu\n",
               sizeof(Key) * 8, K, NW, (int)Second, mode, i, i / K, i % K, (unsigned long long)got[i],
               (unsigned long long)ref[i]);
        return 1;
    }
    return 0;
}

template <typename Key, int K, int NW>
int both() {
    int f = 0;
    for (int mode = 0; mode < 4; ++mode)
        f += run<Key, K, NW, false>(mode) + run<Key, K, NW, true>(mode) + run<Key, K, NW, false, false>(mode) +
             run<Key, K, NW, true, false>(mode);
    return f;
}

int main(int argc, char** argv) {
    int f = 0;
    if (argc > 1) {  // replay a dumped failing input pair (2K u32 keys)
        static uint32_t buf[2048];
        FILE* fp = fopen(argv[1], "rb");
        if (!fp || fread(buf, 4, 2048, fp) != 2048) { printf("bad replay file\n"); return 2; }
        fclose(fp);
        replay_buf = buf;
        f += run<uint32_t, 1024, 4, true, false>(4) + run<uint32_t, 1024, 4, true, true>(4) + run<uint32_t, 1024, 16, true, false>(4);
        printf("replay: %s\n", f ? "FAIL" : "ok");
        return f != 0;
    }
    f += both<uint32_t, 16, 1>();
    f += both<uint32_t, 32, 1>() + both<uint32_t, 32, 4>();
    f += both<uint32_t, 64, 1>() + both<uint32_t, 64, 2>();
    f += both<uint32_t, 128, 1>() + both<uint32_t, 128, 4>();
    f += both<uint32_t, 256, 1>() + both<uint32_t, 256, 2>() + both<uint32_t, 256, 4>() + both<uint32_t, 256, 8>();
    f += both<uint32_t, 512, 2>() + both<uint32_t, 512, 4>() + both<uint32_t, 512, 8>();
    f += both<uint32_t, 1024, 4>() + both<uint32_t, 1024, 8>() + both<uint32_t, 1024, 16>();
    f += both<uint32_t, 2048, 4>() + both<uint32_t, 2048, 8>() + both<uint32_t, 2048, 16>() + both<uint32_t, 2048, 2>();
    f += both<unsigned long long, 1024, 4>() + both<unsigned long long, 1024, 16>() + both<unsigned long long, 256, 1>();
    f += both<unsigned long long, 2048, 8>() + both<unsigned long long, 32, 1>();
    printf("bt_check: %s (%d failing cases)\n", f ? "FAIL" : "ok", f);
    return f != 0;
}

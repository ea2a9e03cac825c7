// Kernel instantiations for 32-bit keys (all node capacities 1..2048).
#include "bh_kernels.cuh"

namespace bh {
using KeyT = uint32_t;
int ops_u32(const HeapView& hv, const RunView& rv, uint32_t ctas, cudaStream_t s) {
    return dispatch_ops<KeyT>(hv, rv, ctas, s);
}
int info_u32(uint32_t k, KernelInfo* info) { return dispatch_info<KeyT>(k, info); }
int sort_u32(uint32_t k, void* keys, const uint32_t* lens, uint64_t rows, cudaStream_t s) {
    return dispatch_sort<KeyT>(k, keys, lens, rows, s);
}
int merge_u32(uint32_t k, const void* a, const void* b, void* hi, void* lo, uint64_t rows, cudaStream_t s) {
    return dispatch_merge<KeyT>(k, a, b, hi, lo, rows, s);
}
int check_u32(const HeapView& hv, unsigned long long* result, cudaStream_t s) {
    return launch_check<KeyT>(hv, result, s);
}
int gather_u32(const HeapView& hv, unsigned long long nodes, void* out, cudaStream_t s) {
    return launch_gather<KeyT>(hv, nodes, out, s);
}
}  // namespace bh

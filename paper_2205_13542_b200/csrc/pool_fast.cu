// pool_fast.cu -- instantiates the interval kernel family: fp32-accumulating reference formulation.
// (Split from pool.cu so the kernel families compile in parallel.)
#include "pool_ivl.cuh"

namespace bvp {

template <>
int run_pool<float, float, 4, kSrcDist>(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    return run_pool_fast<float, 4, kSrcDist>(p, B, is_max, s);
}

template <>
int run_pool<float, float, 1, kSrcDist>(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    return run_pool_fast<float, 1, kSrcDist>(p, B, is_max, s);
}

}  // namespace bvp

using namespace bvp;

extern "C" int bvp_pool_needs_units(int C, int bf16, int exact) {
    (void)exact;  // both modes run on the chunk schedule when the width fits
    const int vec = bf16 ? (C % 8 == 0 ? 8 : 1) : (C % 4 == 0 ? 4 : 1);
    int L, lg, cpl;
    return choose_group(C / vec, vec, L, lg, cpl) ? 0 : 1;
}

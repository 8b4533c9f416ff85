// pool_x.cu -- instantiates the interval kernel family: materialised frustum rows.
// (Split from pool.cu so the kernel families compile in parallel.)
#include "pool_ivl.cuh"

namespace bvp {

template <>
int run_pool<float, float, 4, kSrcX>(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    return run_pool_fast<float, 4, kSrcX>(p, B, is_max, s);
}

template <>
int run_pool<float, float, 1, kSrcX>(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    return run_pool_fast<float, 1, kSrcX>(p, B, is_max, s);
}

}  // namespace bvp

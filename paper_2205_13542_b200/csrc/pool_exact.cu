// pool_exact.cu -- instantiates the interval kernel family: 64-bit bit-exact reference formulation.
// (Split from pool.cu so the kernel families compile in parallel.)
#include "pool_ivl.cuh"

namespace bvp {

template <>
int run_pool<double, float, 4, kSrcDist>(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    const int rc = run_pool_ivl<float, 4, kSrcDist, true>(p, B, is_max, s);
    return rc != BVP_ERR_UNSUPPORTED ? rc : run_pool_ref<float, kSrcDist>(p, B, is_max, s);
}

template <>
int run_pool<double, float, 1, kSrcDist>(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    const int rc = run_pool_ivl<float, 1, kSrcDist, true>(p, B, is_max, s);
    return rc != BVP_ERR_UNSUPPORTED ? rc : run_pool_ref<float, kSrcDist>(p, B, is_max, s);
}

}  // namespace bvp

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

// Zero fill of the empty cells of out (B, C, n_cells): the cells no interval
// covers (cell_first[c] == cell_first[c+1]).  Occupied cells are left as they are.
extern "C" int bvp_zero_empty_cells(const uint32_t *cell_first, int64_t n_cells, int C, int B,
                                    float *out, void *stream) {
    BVP_REQUIRE(n_cells >= 0 && C >= 0 && B >= 0, BVP_ERR_INVALID, "bad dims");
    if (n_cells == 0 || C == 0 || B == 0) return BVP_OK;
    BVP_REQUIRE(cell_first && out, BVP_ERR_INVALID, "null pointer argument");
    bvp::zero_empty_cells_kernel<<<bvp::kNumSms, bvp::kZeroThreads, 0,
                                   static_cast<cudaStream_t>(stream)>>>(cell_first, n_cells, C, B,
                                                                         out);
    return bvp::check_launch("zero_empty_cells");
}

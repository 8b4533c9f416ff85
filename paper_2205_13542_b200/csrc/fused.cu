// fused.cu -- config F: lift + pool fused, bf16 inputs, fp32 accumulation.
//
// The frustum tensor x = softmax_D(logits) (x) context is never formed: a
// small prologue computes each pixel's log-sum-exp over D (N*H*W floats) and
// the NHWC bf16 copy of the context; the interval kernel then forms
// exp(logit - lse) * context[c] in registers per point (pool_kernel.cuh,
// kSrcFused).  Reference semantics: normalize_depth (lift.py:17-31) followed
// by pool_interval (pooling.py:206-221).
#include <algorithm>

#include "pool_kernel.cuh"

namespace bvp {

template <typename T>
void launch_to_nhwc(const T *src, int64_t NB, int A, int HW, T *dst, cudaStream_t s);

// lse[pix] = max_d l + log(sum_d exp(l - max)); thread per pixel, the D
// loads of consecutive pixels are coalesced.
__global__ void pixel_lse_kernel(const __nv_bfloat16 *__restrict__ logits, int64_t NB, int D,
                                 int HW, float *__restrict__ lse) {
    const int64_t total = NB * HW;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = t / HW, hw = t - n * HW;
        const __nv_bfloat16 *l = logits + n * D * int64_t(HW) + hw;
        float m = -INFINITY;
        for (int d = 0; d < D; ++d) m = fmaxf(m, __bfloat162float(l[int64_t(d) * HW]));
        float s = 0.f;
        for (int d = 0; d < D; ++d) s += __expf(__bfloat162float(l[int64_t(d) * HW]) - m);
        lse[t] = m + __logf(s);
    }
}

template <int VEC, int SRC>
struct BfTable;

#define BVP_SHAPE(L, CP)                                                                   \
    if (sh.lpp == L && sh.cpl == CP) {                                                     \
        auto k = is_max ? pool_tile_kernel<float, __nv_bfloat16, VEC, L, CP, true, SRC>    \
                        : pool_tile_kernel<float, __nv_bfloat16, VEC, L, CP, false, SRC>;  \
        if (smem > 48 * 1024)                                                              \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        k<<<grid, kPoolThreads, smem, s>>>(p);                                             \
        return true;                                                                       \
    }

template <int SRC>
struct BfTable<8, SRC> {
    static constexpr int VEC = 8;
    static bool launch(LaneShape sh, const PoolParams &p, bool is_max, dim3 grid, size_t smem,
                       cudaStream_t s) {
        BVP_SHAPE(1, 1) BVP_SHAPE(2, 1) BVP_SHAPE(2, 2) BVP_SHAPE(2, 3) BVP_SHAPE(2, 4)
        BVP_SHAPE(2, 5) BVP_SHAPE(8, 8) BVP_SHAPE(16, 8) BVP_SHAPE(32, 8)
        return false;
    }
};
template <int SRC>
struct BfTable<1, SRC> {
    static constexpr int VEC = 1;
    static bool launch(LaneShape sh, const PoolParams &p, bool is_max, dim3 grid, size_t smem,
                       cudaStream_t s) {
        BVP_SHAPE(32, 1) BVP_SHAPE(32, 2) BVP_SHAPE(32, 4) BVP_SHAPE(32, 8)
        return false;
    }
};
#undef BVP_SHAPE

struct FusedLayout {
    size_t off_lse, off_ctx, bytes;
};
static FusedLayout fused_layout(int B, int N, int C, int H, int W) {
    FusedLayout L{};
    const size_t npix = size_t(B) * N * H * W;
    L.off_lse = 0;
    L.off_ctx = (npix * sizeof(float) + 255) & ~size_t(255);
    L.bytes = L.off_ctx + npix * C * sizeof(__nv_bfloat16);
    return L;
}

}  // namespace bvp

using namespace bvp;

extern "C" {

size_t bvp_fused_workspace_bytes(int B, int N, int C, int H, int W) {
    return fused_layout(B, N, C, H, W).bytes;
}

int bvp_fused_pool_bf16(const uint16_t *logits, const uint16_t *context, const uint32_t *ranks,
                        const uint32_t *interval_starts, const uint32_t *interval_cells,
                        const uint32_t *tile_first, int B, int N, int C, int H, int W, int D,
                        int64_t n_cells, int mode, float *out, void *workspace,
                        size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(B >= 1 && N >= 1 && C >= 0 && H >= 1 && W >= 1 && D >= 1 && n_cells >= 1,
                BVP_ERR_INVALID, "bad dims");
    BVP_REQUIRE(mode >= 0 && mode <= 2, BVP_ERR_INVALID, "bad mode %d", mode);
    const FusedLayout L = fused_layout(B, N, C, H, W);
    BVP_REQUIRE(workspace && workspace_bytes >= L.bytes, BVP_ERR_INVALID,
                "fused workspace too small: need %zu bytes", L.bytes);
    BVP_REQUIRE(out && logits && (C == 0 || (context && ranks && interval_starts &&
                                             interval_cells && tile_first)),
                BVP_ERR_INVALID, "null pointer argument");
    if (C == 0) return BVP_OK;
    cudaStream_t s = as_stream(stream);
    char *ws = static_cast<char *>(workspace);
    float *lse = reinterpret_cast<float *>(ws + L.off_lse);
    auto *ctx = reinterpret_cast<__nv_bfloat16 *>(ws + L.off_ctx);
    const int64_t NB = int64_t(B) * N, HW = int64_t(H) * W;
    const unsigned lb = static_cast<unsigned>(std::min<int64_t>(ceil_div(NB * HW, 128), 148 * 16));
    auto *lg = reinterpret_cast<const __nv_bfloat16 *>(logits);
    pixel_lse_kernel<<<lb, 128, 0, s>>>(lg, NB, D, int(HW), lse);
    launch_to_nhwc<__nv_bfloat16>(reinterpret_cast<const __nv_bfloat16 *>(context), NB, C,
                                  int(HW), ctx, s);
    PoolParams p{};
    p.rows = ctx;
    p.wsrc = lg;
    p.lse = lse;
    p.ranks = ranks;
    p.starts = interval_starts;
    p.icells = interval_cells;
    p.tile_first = tile_first;
    p.out = out;
    p.C = C;
    p.D = D;
    p.HW = int(HW);
    p.NHW = int(N * HW);
    p.mean = mode == BVP_MEAN;
    p.n_cells = n_cells;
    p.rows_bstride = int64_t(N) * HW * C;
    p.w_bstride = int64_t(N) * D * HW;
    const bool is_max = mode == BVP_MAX;
    const bool v8 = (C % 8) == 0;
    const LaneShape sh = choose_shape(v8 ? C / 8 : C, !v8, v8);
    BVP_REQUIRE(sh.lpp > 0, BVP_ERR_UNSUPPORTED, "channel count %d not supported", C);
    const size_t smem = size_t(C) * kTilePitch * sizeof(float);
    BVP_REQUIRE(smem <= 227 * 1024, BVP_ERR_UNSUPPORTED, "channel count %d too large", C);
    const dim3 grid(static_cast<unsigned>(ceil_div(n_cells, kTileCells)), static_cast<unsigned>(B));
    const bool ok = v8 ? BfTable<8, kSrcFused>::launch(sh, p, is_max, grid, smem, s)
                       : BfTable<1, kSrcFused>::launch(sh, p, is_max, grid, smem, s);
    BVP_REQUIRE(ok, BVP_ERR_UNSUPPORTED, "no kernel instance for lpp=%d cpl=%d", sh.lpp, sh.cpl);
    return check_launch("fused_pool_bf16");
}

}  // extern "C"

// pool.cu -- cached-forward entry points (reference formulation and the
// materialised frustum), layout transposes, depth softmax, reorder_weights,
// finiteness scan.  The interval kernels themselves are pool_kernel.cuh,
// instantiated in pool_fast.cu / pool_exact.cu / pool_x.cu.
//
// Reference: pooling.py:206-221 (pool_interval), _kernels.py:22-63
// (interval_reduce), pooling.py:243-261 (reorder_weights), lift.py:17-31
// (normalize_depth), pooling.py:92-95 (finiteness checks).
#include <algorithm>

#include "pool_kernel.cuh"

namespace bvp {

// ---- (N, A, HW) -> (N, HW, A) transpose through a 32x32 shared tile --------
template <typename T>
__global__ void __launch_bounds__(256)
to_nhwc_kernel(const T *__restrict__ src, int A, int HW, T *__restrict__ dst) {
    __shared__ T t[32][33];
    const int64_t n = blockIdx.z;
    const int hw0 = blockIdx.x * 32, a0 = blockIdx.y * 32;
    const T *s = src + n * int64_t(A) * HW;
    T *d = dst + n * int64_t(A) * HW;
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int a = a0 + r, hw = hw0 + threadIdx.x;
        if (a < A && hw < HW) t[r][threadIdx.x] = s[int64_t(a) * HW + hw];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int hw = hw0 + r, a = a0 + threadIdx.x;
        if (a < A && hw < HW) d[int64_t(hw) * A + a] = t[threadIdx.x][r];
    }
}

// Whole-row variant (A <= kRowsA): a CTA moves 32 pixels x all A channels;
// the loads are 128-byte rows of one channel, the stores one contiguous
// 32 x A block of the NHWC output (A * 128 bytes), written as 16-byte words.
constexpr int kRowsA = 128;
template <typename T>
__global__ void __launch_bounds__(256)
to_nhwc_rows_kernel(const T *__restrict__ src, int A, int HW, T *__restrict__ dst) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    T *t = reinterpret_cast<T *>(s_raw);  // [32][A + pad] (pixel-major)
    const int pitch = A + (16 / int(sizeof(T)));
    const int64_t n = blockIdx.y;
    const int hw0 = blockIdx.x * 32;
    const int np = min(32, HW - hw0);
    const T *sb = src + n * int64_t(A) * HW + hw0;
    // every load of the tile issued before the first shared store (A <= 128:
    // <= 16 per thread), so a block waits one memory latency, not A / 8
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T v[kRowsA / 8];
#pragma unroll
    for (int i = 0; i < kRowsA / 8; ++i) {
        const int a = w + 8 * i;
        if (a < A && lane < np) v[i] = sb[int64_t(a) * HW + lane];
    }
#pragma unroll
    for (int i = 0; i < kRowsA / 8; ++i) {
        const int a = w + 8 * i;
        if (a < A && lane < np) t[lane * pitch + a] = v[i];
    }
    __syncthreads();
    T *db = dst + (n * HW + hw0) * int64_t(A);
    constexpr int V = 16 / sizeof(T);
    const int total = np * A;  // contiguous in the output
    if ((A % V) == 0) {
        for (int e = threadIdx.x * V; e < total; e += 256 * V) {
            const int px = e / A, a = e - px * A;
            *reinterpret_cast<uint4 *>(db + e) = *reinterpret_cast<const uint4 *>(t + px * pitch + a);
        }
    } else {
        for (int e = threadIdx.x; e < total; e += 256) {
            const int px = e / A, a = e - px * A;
            db[e] = t[px * pitch + a];
        }
    }
}

template <typename T>
void launch_to_nhwc(const T *src, int64_t NB, int A, int HW, T *dst, cudaStream_t s) {
    if (NB == 0 || A == 0 || HW == 0) return;
    if (A <= kRowsA) {
        const size_t smem = size_t(32) * (A + 16 / sizeof(T)) * sizeof(T);
        const dim3 grid((HW + 31) / 32, static_cast<unsigned>(NB));
        to_nhwc_rows_kernel<T><<<grid, 256, smem, s>>>(src, A, HW, dst);
        return;
    }
    const dim3 grid((HW + 31) / 32, (A + 31) / 32, static_cast<unsigned>(NB));
    to_nhwc_kernel<T><<<grid, dim3(32, 8), 0, s>>>(src, A, HW, dst);
}
template void launch_to_nhwc<float>(const float *, int64_t, int, int, float *, cudaStream_t);
template void launch_to_nhwc<__nv_bfloat16>(const __nv_bfloat16 *, int64_t, int, int,
                                            __nv_bfloat16 *, cudaStream_t);

PoolParams make_pool_params(const uint32_t *ranks, const uint32_t *starts, const uint32_t *icells,
                            const uint32_t *cell_first, const bvp_schedule *sched, int C, int nx,
                            int ny, float *out, int mode) {
    PoolParams p{};
    p.ranks = ranks;
    p.starts = starts;
    p.icells = icells;
    p.cell_first = cell_first;
    p.meta = reinterpret_cast<const uint2 *>(sched->point_meta);
    p.work = reinterpret_cast<const uint4 *>(sched->work);
    p.splits = reinterpret_cast<const uint4 *>(sched->splits);
    p.work_counts = sched->work_counts;
    p.max_work = sched->max_work;
    p.max_splits = sched->max_splits;
    p.chunk_partials = sched->max_partials;
    p.chunk = static_cast<int>(sched->chunk);
    p.out = out;
    p.C = C;
    p.nx = nx;
    p.ny = ny;
    p.n_cells = int64_t(nx) * ny;
    p.mean = mode == BVP_MEAN ? 1 : mode == BVP_MEAN_DIV ? 2 : 0;
    return p;
}

// ---- depth softmax (lift.py:17-31), 64-bit math ------------------------------
// Thread per pixel, the depth bins in order (any D).
__global__ void normalize_depth_kernel(const float *__restrict__ logits, int64_t NB, int D,
                                       int HW, float *__restrict__ dist) {
    const int64_t total = NB * HW;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = t / HW, hw = t - n * HW;
        const float *l = logits + n * D * int64_t(HW) + hw;
        float *o = dist + n * D * int64_t(HW) + hw;
        float m = -INFINITY;
        for (int d = 0; d < D; ++d) m = fmaxf(m, l[int64_t(d) * HW]);
        double sum = 0.0;
        for (int d = 0; d < D; ++d) sum += exp(double(l[int64_t(d) * HW]) - double(m));
        for (int d = 0; d < D; ++d)
            o[int64_t(d) * HW] = float(exp(double(l[int64_t(d) * HW]) - double(m)) / sum);
    }
}

// D <= 8 * kSoftSlice: CTA per 32 pixels (lane = pixel, coalesced), warp w
// owns the contiguous depth slice [w*S, (w+1)*S): its logits and their fp64
// exponentials stay in registers (one exp per point), the slice sums are
// added in slice order -- so every pixel's sum runs over d in order, in 8
// sequential pieces.
constexpr int kSoftSlice = 16;
__global__ void __launch_bounds__(256)
normalize_depth_tile_kernel(const float *__restrict__ logits, int64_t NB, int D, int HW,
                            float *__restrict__ dist) {
    __shared__ float s_m[8][32];
    __shared__ double s_s[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tiles = (HW + 31) / 32;
    const int64_t n = blockIdx.x / tiles;
    const int hw = int(blockIdx.x - n * tiles) * 32 + lane;
    const bool ok = hw < HW;
    const int S = (D + 7) / 8, d0 = warp * S, d1 = min(D, d0 + S);
    const float *l = logits + n * D * int64_t(HW) + (ok ? hw : 0);
    float v[kSoftSlice];
    float m = -INFINITY;
#pragma unroll
    for (int i = 0; i < kSoftSlice; ++i) {
        v[i] = (d0 + i < d1) ? l[int64_t(d0 + i) * HW] : -INFINITY;
        m = fmaxf(m, v[i]);
    }
    s_m[warp][lane] = m;
    __syncthreads();
    float M = s_m[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) M = fmaxf(M, s_m[w][lane]);
    double e[kSoftSlice];
    double part = 0.0;
#pragma unroll
    for (int i = 0; i < kSoftSlice; ++i) {
        e[i] = (d0 + i < d1) ? exp(double(v[i]) - double(M)) : 0.0;
        part += e[i];
    }
    s_s[warp][lane] = part;
    __syncthreads();
    double sum = s_s[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) sum += s_s[w][lane];
    if (!ok) return;
    float *o = dist + n * D * int64_t(HW) + hw;
#pragma unroll
    for (int i = 0; i < kSoftSlice; ++i)
        if (d0 + i < d1) o[int64_t(d0 + i) * HW] = float(e[i] / sum);
}

__global__ void any_nonfinite_kernel(const float *__restrict__ x, int64_t n, int *flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void reorder_weights_kernel(const float *__restrict__ dist,
                                       const uint32_t *__restrict__ ranks, int64_t n_in, int D,
                                       int HW, float *__restrict__ w) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_in;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = ranks[j];
        const uint32_t pix = p / D, d = p - pix * D;
        const uint32_t n = pix / HW, hw = pix - n * HW;
        w[j] = __ldg(dist + (int64_t(n) * D + d) * HW + hw);
    }
}

// ---- materialised lift: x[(pix*D + d), c] = dist[n,d,h,w] * f[n,c,h,w] -----
// One warp per pixel; the pixel's feature column (NCHW, strided) and depth
// weights are staged in shared memory, then its D x C block of x --
// contiguous in the reference point order -- is streamed as flat float4s
// (fully coalesced, evict-first stores).
__global__ void __launch_bounds__(256)
lift_kernel(const float *__restrict__ features, const float *__restrict__ dist, int64_t NP,
            int C, int D, int HW, float *__restrict__ x) {
    extern __shared__ float sm[];  // per warp: C + D floats
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *sf = sm + warp * (C + D);
    float *sw = sf + C;
    for (int64_t pix = blockIdx.x * 8LL + warp; pix < NP; pix += gridDim.x * 8LL) {
        const int64_t n = pix / HW, hw = pix - n * HW;
        __syncwarp();
        for (int c = lane; c < C; c += 32) sf[c] = features[(n * C + c) * HW + hw];
        for (int d = lane; d < D; d += 32) sw[d] = dist[(n * D + d) * HW + hw];
        __syncwarp();
        float *xo = x + pix * int64_t(D) * C;
        const int n4 = (D * C) / 4;
        for (int q = lane; q < n4; q += 32) {
            const int e = q * 4;
            const int d = e / C, c = e - d * C;  // C % 4 == 0: one depth bin per float4
            const float w = sw[d];
            st_stream_f4(xo + e,
                         make_float4(w * sf[c], w * sf[c + 1], w * sf[c + 2], w * sf[c + 3]));
        }
    }
}

__global__ void lift_scalar_kernel(const float *__restrict__ features,
                                   const float *__restrict__ dist, int64_t NP, int C, int D,
                                   int HW, float *__restrict__ x) {
    const int64_t total = NP * D * int64_t(C);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e % C, pd = e / C;
        const int64_t d = pd % D, pix = pd / D;
        const int64_t n = pix / HW, hw = pix - n * HW;
        x[e] = dist[(n * D + d) * HW + hw] * features[(n * C + c) * HW + hw];
    }
}

}  // namespace bvp

using namespace bvp;

extern "C" {

size_t bvp_pool_scratch_bytes(const bvp_schedule *schedule, int B, int C, int mode) {
    if (!schedule || !schedule->work || schedule->max_splits <= 0) return 0;
    return size_t(B) * schedule->max_partials * C * (mode == BVP_MAX ? 8 : 4);
}

size_t bvp_pool_workspace_bytes(int B, int N, int C, int H, int W) {
    return size_t(B) * N * C * H * W * sizeof(float);
}

int bvp_to_nhwc_f32(const float *src, int NB, int C, int HW, float *dst, void *stream) {
    BVP_REQUIRE(NB >= 0 && C >= 0 && HW >= 0, BVP_ERR_INVALID, "bad dims");
    BVP_REQUIRE((src && dst) || NB * int64_t(C) * HW == 0, BVP_ERR_INVALID,
                "null pointer argument");
    launch_to_nhwc<float>(src, NB, C, HW, dst, as_stream(stream));
    return check_launch("to_nhwc");
}

}  // extern "C"

namespace bvp {
static int pool_forward_nhwc(const float *feats_nhwc, const float *dist, const uint32_t *ranks,
                              const uint32_t *interval_starts, const uint32_t *interval_cells,
                              const uint32_t *cell_first, const bvp_schedule *schedule, int B,
                              int N, int C, int H, int W, int D, int nx, int ny,
                              int64_t n_int_max, int mode, int exact, float *out,
                              uint32_t *argmax, void *scratch, size_t scratch_bytes,
                              void *stream, bool zeroed) {
    BVP_REQUIRE(B >= 1 && N >= 1 && C >= 0 && H >= 1 && W >= 1 && D >= 1 && nx >= 1 && ny >= 1,
                BVP_ERR_INVALID, "bad dims B=%d N=%d C=%d H=%d W=%d D=%d nx=%d ny=%d", B, N, C,
                H, W, D, nx, ny);
    BVP_REQUIRE(mode >= 0 && mode <= 2 || (mode == BVP_MEAN_DIV && exact), BVP_ERR_INVALID,
                "bad mode %d", mode);
    BVP_REQUIRE(C == 0 || (out && feats_nhwc && dist && ranks && interval_starts &&
                           interval_cells && cell_first && schedule),
                BVP_ERR_INVALID, "null pointer argument");
    if (C == 0) return BVP_OK;
    PoolParams p = make_pool_params(ranks, interval_starts, interval_cells, cell_first, schedule,
                                    C, nx, ny, out, mode);
    p.rows = feats_nhwc;
    p.wsrc = dist;
    p.argmax = mode == BVP_MAX ? argmax : nullptr;
    p.D = D;
    p.HW = H * W;
    p.NHW = N * H * W;
    p.n_int_max = n_int_max;
    p.rows_bstride = int64_t(N) * H * W * C;
    p.w_bstride = int64_t(N) * D * H * W;
    p.scratch = scratch;
    p.scratch_bytes = scratch_bytes;
    p.out_zeroed = zeroed ? 1 : 0;
    const bool is_max = mode == BVP_MAX, v4 = (C % 4) == 0;
    cudaStream_t s = as_stream(stream);
    int rc;
    if (exact)
        rc = v4 ? run_pool<double, float, 4, kSrcDist>(p, B, is_max, s)
                : run_pool<double, float, 1, kSrcDist>(p, B, is_max, s);
    else
        rc = v4 ? run_pool<float, float, 4, kSrcDist>(p, B, is_max, s)
                : run_pool<float, float, 1, kSrcDist>(p, B, is_max, s);
    if (rc != BVP_OK) return rc;
    return check_launch("pool_forward");
}
}  // namespace bvp

extern "C" {

int bvp_pool_forward_nhwc_f32(const float *feats_nhwc, const float *dist, const uint32_t *ranks,
                              const uint32_t *interval_starts, const uint32_t *interval_cells,
                              const uint32_t *cell_first, const bvp_schedule *schedule, int B,
                              int N, int C, int H, int W, int D, int nx, int ny,
                              int64_t n_int_max, int mode, int exact, float *out,
                              uint32_t *argmax, void *scratch, size_t scratch_bytes,
                              void *stream) {
    return pool_forward_nhwc(feats_nhwc, dist, ranks, interval_starts, interval_cells,
                             cell_first, schedule, B, N, C, H, W, D, nx, ny, n_int_max,
                             mode & ~BVP_OUT_ZEROED, exact, out, argmax, scratch, scratch_bytes,
                             stream, (mode & BVP_OUT_ZEROED) != 0);
}

int bvp_pool_prepare_f32(const float *features, int B, int N, int C, int H, int W,
                         float *feats_nhwc, float *out, int64_t n_cells, void *stream) {
    BVP_REQUIRE(B >= 1 && N >= 1 && C >= 0 && H >= 1 && W >= 1 && n_cells >= 1,
                BVP_ERR_INVALID, "bad dims");
    BVP_REQUIRE(C == 0 || (features && feats_nhwc), BVP_ERR_INVALID, "null pointer argument");
    if (C == 0) return BVP_OK;
    cudaStream_t s = as_stream(stream);
    if (!out) {  // no zero fill: the reduction zeroes the empty cells beside its kernels
        launch_to_nhwc<float>(features, int64_t(B) * N, C, H * W, feats_nhwc, s);
        return check_launch("pool_prepare");
    }
    // the map's zero fill (for the chunk kernel's scattered column stores)
    // runs beside the features' NHWC transpose: two graph branches
    SideFork fork(s);
    cudaMemsetAsync(out, 0, size_t(B) * C * n_cells * sizeof(float), fork.side);
    launch_to_nhwc<float>(features, int64_t(B) * N, C, H * W, feats_nhwc, s);
    fork.join();
    return check_launch("pool_prepare");
}

int bvp_pool_forward_f32(const float *features, const float *dist, const uint32_t *ranks,
                         const uint32_t *interval_starts, const uint32_t *interval_cells,
                         const uint32_t *cell_first, const bvp_schedule *schedule, int B, int N,
                         int C, int H, int W, int D, int nx, int ny, int64_t n_int_max, int mode,
                         int exact, float *out, float *feats_nhwc, uint32_t *argmax,
                         void *scratch, size_t scratch_bytes, void *stream) {
    BVP_REQUIRE(B >= 1 && N >= 1 && C >= 0 && H >= 1 && W >= 1, BVP_ERR_INVALID, "bad dims");
    BVP_REQUIRE(C == 0 || (features && feats_nhwc && out), BVP_ERR_INVALID,
                "null pointer argument");
    if (C == 0) return BVP_OK;
    // the memset of the map beside the NHWC transpose, then the reduction
    const int rc = bvp_pool_prepare_f32(features, B, N, C, H, W, feats_nhwc, out,
                                        int64_t(nx) * ny, stream);
    if (rc != BVP_OK) return rc;
    return pool_forward_nhwc(feats_nhwc, dist, ranks, interval_starts, interval_cells, cell_first,
                             schedule, B, N, C, H, W, D, nx, ny, n_int_max, mode, exact, out,
                             argmax, scratch, scratch_bytes, stream, true);
}

int bvp_reorder_weights(const float *dist, const uint32_t *ranks, int64_t n_in, int N, int D,
                        int H, int W, float *w_sorted, void *stream) {
    BVP_REQUIRE(n_in == 0 || (dist && ranks && w_sorted), BVP_ERR_INVALID, "null pointer");
    (void)N;
    if (n_in == 0) return BVP_OK;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(n_in, 256), 148 * 32));
    reorder_weights_kernel<<<blocks, 256, 0, as_stream(stream)>>>(dist, ranks, n_in, D, H * W,
                                                                  w_sorted);
    return check_launch("reorder_weights");
}

int bvp_normalize_depth(const float *logits, int NB, int D, int H, int W, float *dist,
                        void *stream) {
    BVP_REQUIRE(logits && dist && NB >= 0 && D >= 1 && H >= 0 && W >= 0, BVP_ERR_INVALID,
                "bad arguments");
    const int64_t total = int64_t(NB) * H * W;
    if (total == 0) return BVP_OK;
    if (D <= 8 * kSoftSlice) {
        const int64_t tiles = int64_t(NB) * ceil_div(int64_t(H) * W, 32);
        normalize_depth_tile_kernel<<<static_cast<unsigned>(tiles), 256, 0, as_stream(stream)>>>(
            logits, NB, D, H * W, dist);
        return check_launch("normalize_depth");
    }
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 128), 148 * 16));
    normalize_depth_kernel<<<blocks, 128, 0, as_stream(stream)>>>(logits, NB, D, H * W, dist);
    return check_launch("normalize_depth");
}

int bvp_any_nonfinite(const float *x, int64_t n, int *flag, void *stream) {
    BVP_REQUIRE(flag && (n == 0 || x), BVP_ERR_INVALID, "null pointer");
    if (n == 0) return BVP_OK;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 148 * 8));
    any_nonfinite_kernel<<<blocks, 256, 0, as_stream(stream)>>>(x, n, flag);
    return check_launch("any_nonfinite");
}

int bvp_lift_f32(const float *features, const float *dist, int N, int C, int H, int W, int D,
                 float *x, void *stream) {
    BVP_REQUIRE(features && dist && x && N >= 1 && C >= 1 && H >= 1 && W >= 1 && D >= 1,
                BVP_ERR_INVALID, "bad arguments");
    cudaStream_t s = as_stream(stream);
    const int64_t NP = int64_t(N) * H * W;
    if (C % 4 == 0) {
        const size_t smem = size_t(8) * (C + D) * sizeof(float);
        BVP_REQUIRE(smem <= 227 * 1024, BVP_ERR_UNSUPPORTED, "C + D too large for lift");
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(lift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem));
        const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(NP, 8), 148 * 16));
        lift_kernel<<<blocks, 256, smem, s>>>(features, dist, NP, C, D, H * W, x);
    } else {
        const int64_t total = NP * D * C;
        const unsigned blocks =
            static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 256), 148 * 64));
        lift_scalar_kernel<<<blocks, 256, 0, s>>>(features, dist, NP, C, D, H * W, x);
    }
    return check_launch("lift");
}

int bvp_pool_lifted_f32(const float *x, const uint32_t *ranks, const uint32_t *interval_starts,
                        const uint32_t *interval_cells, const uint32_t *cell_first,
                        const bvp_schedule *schedule, int C, int nx, int ny, int mode,
                        float *out, void *scratch, size_t scratch_bytes, void *stream) {
    BVP_REQUIRE(C >= 0 && nx >= 1 && ny >= 1 && mode >= 0 && mode <= 2, BVP_ERR_INVALID,
                "bad arguments");
    BVP_REQUIRE(C == 0 || (out && x && ranks && interval_starts && interval_cells && cell_first &&
                           schedule),
                BVP_ERR_INVALID, "null pointer argument");
    if (C == 0) return BVP_OK;
    PoolParams p = make_pool_params(ranks, interval_starts, interval_cells, cell_first, schedule,
                                    C, nx, ny, out, mode);
    p.rows = x;
    p.D = 1;
    p.HW = 1;
    p.scratch = scratch;
    p.scratch_bytes = scratch_bytes;
    const bool is_max = mode == BVP_MAX;
    cudaStream_t s = as_stream(stream);
    const int rc = (C % 4 == 0) ? run_pool<float, float, 4, kSrcX>(p, 1, is_max, s)
                                : run_pool<float, float, 1, kSrcX>(p, 1, is_max, s);
    if (rc != BVP_OK) return rc;
    return check_launch("pool_lifted");
}

}  // extern "C"

// backward.cu -- gather backward of the interval pooling (config B).
//
// The reference has no backward (SPEC.md:540 lists autograd as a non-goal);
// the math is the adjoint of pool_interval (pooling.py:206-221):
//   out[c, cell] = red_{p in cell} w_p * f[pix(p), c]
//   SUM : dL/dv_p = g[:, cell(p)]        MEAN: ... / len(cell)
//   MAX : g[c, cell] routed to the winning point of (cell, c) (first in rank
//         order, recorded by the forward as `argmax`)
//   grad_f[n,c,h,w] = sum_d w_p dL/dv_p[c],  grad_w[n,d,h,w] = <f[pix], dL/dv_p>
//
// No atomics: step 1 turns grad_out (C, n_cells) into per-interval rows
// gT[i, :] (scaled for MEAN) through a coalesced shared-memory transpose; step
// 2 walks the frustum in POINT order -- one warp per pixel, its D points'
// interval ids are contiguous in interval_of_point -- gathering gT rows, so
// every gradient element is produced by exactly one warp.  The 32 per-point
// dot products of a depth block are reduced with a 31-shuffle transpose-
// reduction instead of 32 separate butterflies.
#include <algorithm>

#include "pool_kernel.cuh"

namespace bvp {

constexpr int kRowPitch = kTileCells + 1;

// CTA per 32-cell row tile (ix, ty), like the forward's warp tiles.
template <bool MEAN>
__global__ void __launch_bounds__(128)
grad_rows_kernel(const float *__restrict__ grad_out, const uint32_t *__restrict__ starts,
                 const uint32_t *__restrict__ icells, const uint32_t *__restrict__ cell_first,
                 int C, int nx, int ny, int64_t n_int_max, float *__restrict__ gT) {
    extern __shared__ float s[];  // [C][kRowPitch]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.y;
    const int tiles_y = (ny + kTileCells - 1) / kTileCells;
    const int ty = blockIdx.x / nx, ix = blockIdx.x - ty * nx;
    const int64_t n_cells = int64_t(nx) * ny;
    const int64_t cell0 = int64_t(ix) * ny + ty * kTileCells;
    const int rem = min(kTileCells, ny - ty * kTileCells);
    (void)tiles_y;
    const uint32_t i0 = cell_first[cell0], i1 = cell_first[cell0 + rem];
    if (i0 == i1) return;
    const float *g = grad_out + int64_t(b) * C * n_cells + cell0;
    // 8 channel rows per warp in flight at a time
    for (int c0 = warp; c0 < C; c0 += 32) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int c = c0 + 4 * q;
            v[q] = (c < C && lane < rem) ? __ldg(g + int64_t(c) * n_cells + lane) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (c0 + 4 * q < C) s[(c0 + 4 * q) * kRowPitch + lane] = v[q];
    }
    __syncthreads();
    for (uint32_t i = i0 + warp; i < i1; i += 4) {
        const int lc = static_cast<int>(icells[i] - cell0);
        const float scale = MEAN ? 1.f / float(starts[i + 1] - starts[i]) : 1.f;
        float *row = gT + (int64_t(b) * n_int_max + i) * C;
        for (int c = lane; c < C; c += 32) row[c] = s[c * kRowPitch + lc] * scale;
    }
}

__device__ __forceinline__ float transpose_reduce32(float (&part)[32], int lane) {
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
        const bool upper = (lane & sft) != 0;
#pragma unroll
        for (int i = 0; i < sft; ++i) {
            const float send = upper ? part[i] : part[i + sft];
            const float keep = upper ? part[i + sft] : part[i];
            part[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, sft);
        }
    }
    return part[0];
}

// grid (ceil(W/32), N*H, B), 256 threads; CTA = 32 pixels of one image row.
template <int Q, bool IS_MAX>
__global__ void __launch_bounds__(256)
pool_backward_kernel(const float *__restrict__ gT, const uint32_t *__restrict__ argT,
                     const float *__restrict__ feats_nhwc, const float *__restrict__ dist,
                     const uint32_t *__restrict__ iop, int N, int C, int H, int W, int D,
                     int64_t n_int_max, float *__restrict__ grad_f, float *__restrict__ grad_w) {
    extern __shared__ float sm[];
    float *s_gf = sm;                       // [C][kRowPitch]
    float *s_gw = sm + C * kRowPitch;       // [D][kRowPitch]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int w0 = blockIdx.x * 32;
    const int nh = blockIdx.y, b = blockIdx.z;
    const int n = nh / H, h = nh - n * H;
    const int HW = H * W;
    const int64_t NHW = int64_t(N) * HW;
    const int64_t P = NHW * D;
    const float *distb = dist + int64_t(b) * N * D * HW;
    for (int wl = warp; wl < 32; wl += 8) {
        const int w = w0 + wl;
        if (w >= W) break;
        const int hw = h * W + w;
        const int64_t pix = int64_t(n) * HW + hw;
        const int64_t p0 = pix * D;
        float f[Q], af[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = lane + 32 * q;
            f[q] = c < C ? __ldg(feats_nhwc + (int64_t(b) * NHW + pix) * C + c) : 0.f;
            af[q] = 0.f;
        }
        for (int d0 = 0; d0 < D; d0 += 32) {
            const int dl = d0 + lane;
            uint32_t iv_l = kOOR;
            float wt_l = 0.f;
            if (dl < D) {
                iv_l = __ldg(iop + p0 + dl);
                wt_l = __ldg(distb + (int64_t(n) * D + dl) * HW + hw);
            }
            float part[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                part[k] = 0.f;
                const uint32_t iv = __shfl_sync(0xFFFFFFFFu, iv_l, k);
                const float wt = __shfl_sync(0xFFFFFFFFu, wt_l, k);
                if (iv != kOOR) {
                    const int64_t rbase = (int64_t(b) * n_int_max + iv) * C;
                    float dot = 0.f;
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        const int c = lane + 32 * q;
                        if (c < C) {
                            float gv = __ldg(gT + rbase + c);
                            if (IS_MAX && __ldg(argT + rbase + c) != uint32_t(p0 + d0 + k))
                                gv = 0.f;
                            af[q] += wt * gv;
                            dot += f[q] * gv;
                        }
                    }
                    part[k] = dot;
                }
            }
            const float gw = transpose_reduce32(part, lane);
            if (dl < D) s_gw[dl * kRowPitch + wl] = gw;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = lane + 32 * q;
            if (c < C) s_gf[c * kRowPitch + wl] = af[q];
        }
    }
    __syncthreads();
    const int nw = min(32, W - w0);
    if (lane < nw) {
        const int64_t hw = int64_t(h) * W + w0 + lane;
        if (grad_f) {
            float *gf = grad_f + (int64_t(b) * N + n) * C * HW + hw;
            for (int c = warp; c < C; c += 8) gf[int64_t(c) * HW] = s_gf[c * kRowPitch + lane];
        }
        if (grad_w) {
            float *gw = grad_w + (int64_t(b) * N + n) * D * HW + hw;
            for (int d = warp; d < D; d += 8) gw[int64_t(d) * HW] = s_gw[d * kRowPitch + lane];
        }
    }
    (void)P;
}

// SUM / MEAN backward, group layout (measured faster, profiles/): a warp
// takes 8 consecutive pixels of the flattened (N, H*W) frustum, one per
// 4-lane group, and walks their D depth points in step.  Per step each group
// gathers its point's gradient row gT[interval] (5 float4 per lane at C = 80),
// accumulates grad_f += w * g and reduces <f, g> over its 4 lanes into
// grad_w.  The 8 groups' grad_w stores (and, at the end, every channel's
// grad_f stores) are 8 consecutive floats.  Interval ids and weights of a
// 4-point window are loaded one lane per point and shuffled, a window ahead.
// Every gradient element is written by exactly one lane: no atomics.
template <int CPL>
#ifndef BVP_BWD_MIN_BLOCKS
#define BVP_BWD_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(256, BVP_BWD_MIN_BLOCKS)
pool_backward_grp_kernel(const float *__restrict__ gT, const float *__restrict__ feats_nhwc,
                         const float *__restrict__ dist, const uint32_t *__restrict__ iop, int N,
                         int C, int HW, int D, int64_t n_int_max, int L, int lg,
                         float *__restrict__ grad_f, float *__restrict__ grad_w) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> lg, li = lane & (L - 1);
    const int G = 32 >> lg;
    const int b = blockIdx.y;
    const int64_t NHW = int64_t(N) * HW;
    const int nch = C / 4;
    const int64_t pix = (int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * G + g;
    const bool valid = pix < NHW;
    const int64_t px = valid ? pix : 0;
    const int64_t n = px / HW, hw = px - n * HW;
    float f[CPL][4], af[CPL][4];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int ch = li + k * L;
        const bool ok = ch < nch;
        const float4 t = ok ? __ldg(reinterpret_cast<const float4 *>(
                                  feats_nhwc + (int64_t(b) * NHW + px) * C) + ch)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        f[k][0] = t.x; f[k][1] = t.y; f[k][2] = t.z; f[k][3] = t.w;
        af[k][0] = af[k][1] = af[k][2] = af[k][3] = 0.f;
    }
    const uint32_t *ip = iop + px * D;
    const float *wp = dist + (int64_t(b) * N + n) * D * HW + hw;
    float *gw = grad_w ? grad_w + (int64_t(b) * N + n) * D * HW + hw : nullptr;
    const float *gTb = gT + int64_t(b) * n_int_max * C;
    // windows of L points: lane li holds point d0 + li's interval and weight;
    // the current and the next window are kept, the one after is in flight
    auto load_win = [&](int d0, uint32_t &iv, float &w) {
        const int d = d0 + li;
        iv = kOOR;
        w = 0.f;
        if (valid && d < D) {
            iv = __ldg(ip + d);
            w = __ldg(wp + int64_t(d) * HW);
        }
    };
    uint32_t iv0, iv1, iv2;
    float w0, w1, w2;
    load_win(0, iv0, w0);
    load_win(L, iv1, w1);
    load_win(2 * L, iv2, w2);
    int wbase = 0;  // first point of window 0
    const int gbase = g * L;
    // point d's (interval, weight): window 0 or 1 (d < wbase + 2L always)
    auto point = [&](int d, uint32_t &iv, float &w) {
        const int q = d - wbase;
        const int src = gbase + (q & (L - 1));
        const uint32_t a0 = __shfl_sync(0xFFFFFFFFu, iv0, src), a1 = __shfl_sync(0xFFFFFFFFu, iv1, src);
        const float b0 = __shfl_sync(0xFFFFFFFFu, w0, src), b1 = __shfl_sync(0xFFFFFFFFu, w1, src);
        iv = q < L ? a0 : a1;
        w = q < L ? b0 : b1;
    };
    // gradient row of point d into registers (zeros when out of range)
    auto fetch = [&](int d, uint32_t &iv, float &w, float4 (&row)[CPL]) {
        point(d, iv, w);
        const float4 *r = reinterpret_cast<const float4 *>(gTb + int64_t(iv == kOOR ? 0u : iv) * C);
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int ch = li + k * L;
            row[k] = (iv != kOOR && ch < nch) ? __ldg(r + ch) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto consume = [&](int d, float w, const float4 (&row)[CPL]) {
        float dot = 0.f;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const float4 t = row[k];
            af[k][0] = fmaf(w, t.x, af[k][0]);
            af[k][1] = fmaf(w, t.y, af[k][1]);
            af[k][2] = fmaf(w, t.z, af[k][2]);
            af[k][3] = fmaf(w, t.w, af[k][3]);
            dot = fmaf(f[k][0], t.x, dot);
            dot = fmaf(f[k][1], t.y, dot);
            dot = fmaf(f[k][2], t.z, dot);
            dot = fmaf(f[k][3], t.w, dot);
        }
        for (int o = 1; o < L; o <<= 1) dot += __shfl_xor_sync(0xFFFFFFFFu, dot, o);
        if (gw && valid && li == 0) gw[int64_t(d) * HW] = dot;
    };
    // advance the windows so that points d and d + 1 are covered
    auto cover = [&](int d) {
        while (d + 1 >= wbase + 2 * L) {
            iv0 = iv1; w0 = w1;
            iv1 = iv2; w1 = w2;
            wbase += L;
            load_win(wbase + 2 * L, iv2, w2);
        }
    };
    float4 ra[CPL], rb[CPL];
    uint32_t ia, ib;
    float wa, wb;
    fetch(0, ia, wa, ra);
#pragma unroll 1
    for (int d = 0; d < D; d += 2) {
        cover(d);
        if (d + 1 < D) fetch(d + 1, ib, wb, rb);
        consume(d, wa, ra);
        if (d + 1 >= D) break;
        cover(d + 1);
        if (d + 2 < D) fetch(d + 2, ia, wa, ra);
        consume(d + 1, wb, rb);
    }
    if (grad_f && valid) {
        float *gf = grad_f + (int64_t(b) * N + n) * C * HW + hw;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int ch = li + k * L;
            if (ch < nch)
#pragma unroll
                for (int x = 0; x < 4; ++x) gf[int64_t(ch * 4 + x) * HW] = af[k][x];
        }
    }
}

template <bool IS_MAX>
__global__ void lifted_backward_kernel(const float *__restrict__ gT,
                                       const uint32_t *__restrict__ argT,
                                       const uint32_t *__restrict__ iop, int C, int64_t P,
                                       float *__restrict__ grad_x) {
    const int64_t total = P * C;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = e / C, c = e - p * C;
        const uint32_t iv = __ldg(iop + p);
        float v = 0.f;
        if (iv != kOOR) {
            v = __ldg(gT + int64_t(iv) * C + c);
            if (IS_MAX && __ldg(argT + int64_t(iv) * C + c) != uint32_t(p)) v = 0.f;
        }
        grad_x[e] = v;
    }
}

static int launch_grad_rows(const float *grad_out, const uint32_t *starts, const uint32_t *icells,
                            const uint32_t *cell_first, int B, int C, int nx, int ny,
                            int64_t n_int_max, bool mean, float *gT, cudaStream_t s) {
    const size_t smem = size_t(C) * kRowPitch * sizeof(float);
    BVP_REQUIRE(smem <= 227 * 1024, BVP_ERR_UNSUPPORTED, "channel count %d too large", C);
    auto k = mean ? grad_rows_kernel<true> : grad_rows_kernel<false>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int tiles_y = (ny + kTileCells - 1) / kTileCells;
    const dim3 grid(static_cast<unsigned>(int64_t(nx) * tiles_y), static_cast<unsigned>(B));
    k<<<grid, 128, smem, s>>>(grad_out, starts, icells, cell_first, C, nx, ny, n_int_max, gT);
    return BVP_OK;
}

}  // namespace bvp

using namespace bvp;

extern "C" {

size_t bvp_backward_workspace_bytes(int B, int C, int64_t n_int_max) {
    return size_t(B) * size_t(n_int_max > 0 ? n_int_max : 1) * C * sizeof(float);
}

int bvp_pool_backward_f32(const float *grad_out, const float *feats_nhwc, const float *dist,
                          const uint32_t *interval_starts, const uint32_t *interval_cells,
                          const uint32_t *cell_first, const uint32_t *interval_of_point,
                          const uint32_t *argmax, int B, int N, int C, int H, int W, int D,
                          int nx, int ny, int64_t n_int_max, int mode, float *grad_features,
                          float *grad_dist, void *workspace, size_t workspace_bytes,
                          void *stream) {
    BVP_REQUIRE(B >= 1 && N >= 1 && C >= 0 && H >= 1 && W >= 1 && D >= 1 && nx >= 1 && ny >= 1,
                BVP_ERR_INVALID, "bad dims");
    BVP_REQUIRE(mode >= 0 && mode <= 2, BVP_ERR_INVALID, "bad mode %d", mode);
    BVP_REQUIRE(mode != BVP_MAX || argmax, BVP_ERR_INVALID, "MAX backward needs argmax");
    const size_t need = bvp_backward_workspace_bytes(B, C, n_int_max);
    BVP_REQUIRE(workspace && workspace_bytes >= need, BVP_ERR_INVALID,
                "backward workspace too small: need %zu bytes", need);
    BVP_REQUIRE(grad_out && feats_nhwc && dist && interval_starts && interval_cells && cell_first &&
                    interval_of_point,
                BVP_ERR_INVALID, "null pointer argument");
    cudaStream_t s = as_stream(stream);
    if (C == 0) {
        if (grad_dist) cudaMemsetAsync(grad_dist, 0, size_t(B) * N * D * H * W * sizeof(float), s);
        return check_launch("pool_backward");
    }
    const int Q = (C + 31) / 32;
    BVP_REQUIRE(Q <= 8, BVP_ERR_UNSUPPORTED, "backward supports C <= 256, got %d", C);
    float *gT = static_cast<float *>(workspace);
    int rc = launch_grad_rows(grad_out, interval_starts, interval_cells, cell_first, B, C, nx, ny,
                              n_int_max, mode == BVP_MEAN, gT, s);
    if (rc != BVP_OK) return rc;
    int L, lg, cpl;
    if (mode != BVP_MAX && C % 4 == 0 && choose_group(C / 4, 4, L, lg, cpl)) {
        const int64_t NHW = int64_t(N) * H * W;
        const int G = 32 >> lg;
        const dim3 grid(static_cast<unsigned>(ceil_div(ceil_div(NHW, G), 8)), static_cast<unsigned>(B));
#define BVP_BWD_GRP(CPLV)                                                                     \
        if (cpl == CPLV)                                                                      \
            pool_backward_grp_kernel<CPLV><<<grid, 256, 0, s>>>(gT, feats_nhwc, dist,         \
                interval_of_point, N, C, H * W, D, n_int_max, L, lg, grad_features, grad_dist);
        BVP_BWD_GRP(1) BVP_BWD_GRP(2) BVP_BWD_GRP(3) BVP_BWD_GRP(4) BVP_BWD_GRP(5) BVP_BWD_GRP(6)
#undef BVP_BWD_GRP
        return check_launch("pool_backward");
    }
    const size_t smem = size_t(C + D) * kRowPitch * sizeof(float);
    BVP_REQUIRE(smem <= 227 * 1024, BVP_ERR_UNSUPPORTED, "C + D too large for the backward");
    const dim3 grid(static_cast<unsigned>((W + 31) / 32), static_cast<unsigned>(N * H),
                    static_cast<unsigned>(B));
    const bool mx = mode == BVP_MAX;
#define BVP_BWD(QQ)                                                                          \
    case QQ: {                                                                               \
        auto k = mx ? pool_backward_kernel<QQ, true> : pool_backward_kernel<QQ, false>;      \
        if (smem > 48 * 1024)                                                                \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        k<<<grid, 256, smem, s>>>(gT, argmax, feats_nhwc, dist, interval_of_point, N, C, H, W, \
                                  D, n_int_max, grad_features, grad_dist);                   \
        break;                                                                               \
    }
    switch (Q) {
        BVP_BWD(1) BVP_BWD(2) BVP_BWD(3) BVP_BWD(4) BVP_BWD(5) BVP_BWD(6) BVP_BWD(7) BVP_BWD(8)
    }
#undef BVP_BWD
    return check_launch("pool_backward");
}

int bvp_pool_lifted_backward_f32(const float *grad_out, const uint32_t *interval_starts,
                                 const uint32_t *interval_cells, const uint32_t *cell_first,
                                 const uint32_t *interval_of_point, int C, int64_t n_points,
                                 int nx, int ny, int64_t n_int_max, int mode, float *grad_x,
                                 void *workspace, size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(C >= 1 && n_points >= 1 && nx >= 1 && ny >= 1 && mode >= 0 && mode <= 1,
                BVP_ERR_INVALID, "bad arguments (lifted backward supports SUM/MEAN)");
    const size_t need = bvp_backward_workspace_bytes(1, C, n_int_max);
    BVP_REQUIRE(workspace && workspace_bytes >= need, BVP_ERR_INVALID,
                "backward workspace too small: need %zu bytes", need);
    BVP_REQUIRE(grad_out && interval_starts && interval_cells && cell_first && interval_of_point &&
                    grad_x,
                BVP_ERR_INVALID, "null pointer argument");
    cudaStream_t s = as_stream(stream);
    float *gT = static_cast<float *>(workspace);
    int rc = launch_grad_rows(grad_out, interval_starts, interval_cells, cell_first, 1, C, nx, ny,
                              n_int_max, mode == BVP_MEAN, gT, s);
    if (rc != BVP_OK) return rc;
    const unsigned blocks =
        static_cast<unsigned>(std::min<int64_t>(ceil_div(n_points * C, 256), 148 * 64));
    lifted_backward_kernel<false><<<blocks, 256, 0, s>>>(gT, nullptr, interval_of_point, C,
                                                         n_points, grad_x);
    return check_launch("pool_lifted_backward");
}

}  // extern "C"

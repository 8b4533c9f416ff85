// tile_backward.cu -- the adjoint of the tiled reduction: config B's
// bvp_tile_backward_f32 and config F's bvp_tile_fused_backward_bf16 (one
// kernel, FU selecting the bf16 / softmax variant).  See tile.cu for the
// forward it inverts.
#include "tile.cuh"

namespace bvp {

// ---- backward (config B): the adjoint of the tiled reduction ----------------
// out[c, cell] = sum_p w_p f[pix(p), c] (SUM; MEAN scales by 1/len(cell)), so
//   grad_f[pix = (n, h, w), c] = sum_{p of the pixel} w_p g[c, cell(p)]
//                              = sum_k A[k, h] G[k, c]   per tile, over segments k
//   grad_w[p]                  = <f[pix(p), :], g[:, cell(p)]> = Dot[k(p), h(p)]
// with A the forward's aggregated weights and G[k, :] = g[:, cell_k] (x 1/len
// for MEAN) -- the same column tiles, groups and weight windows as the
// forward, so every gradient row is read once per (segment, tile) instead of
// once per point.  No atomics: each gradient element is written once.

// G rows per segment slot: rows[s, :] = g[:, cell(s)] (x 1/len for MEAN), one
// CTA per 32 cells (coalesced channel lines in, a shared-memory transpose,
// 4C-byte rows out); blocks without segments are skipped.
template <int CS>
__global__ void __launch_bounds__(kPoolThreads)
tile_grad_rows_kernel(const float *__restrict__ grad_out, const uint32_t *__restrict__ cell_seg_first,
                      const uint32_t *__restrict__ cell_npts, int n_cells, int C, int mean,
                      int64_t max_seg, float *__restrict__ rows) {
    constexpr int CP = CS * 32;
    constexpr int NW = kPoolThreads / 32;
    __shared__ float tile[CP][kFinCells + 1];
    const int c0 = blockIdx.x * kFinCells, b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nc = min(kFinCells, n_cells - c0);
    const uint32_t f = __ldg(cell_seg_first + c0 + min(lane, nc));
    const uint32_t f_end = __ldg(cell_seg_first + c0 + nc);
    if (__shfl_sync(0xFFFFFFFFu, f, 0) == f_end) return;  // no segment in the block
    const float *gb = grad_out + int64_t(b) * C * n_cells + c0;
#pragma unroll
    for (int k = 0; k < CP / NW; ++k) {
        const int ch = warp + NW * k;
        tile[ch][lane] = ch < C && lane < nc ? __ldg(gb + int64_t(ch) * n_cells + lane) : 0.f;
    }
    __syncthreads();
    float *rb = rows + int64_t(b) * max_seg * C + lane;
#pragma unroll
    for (int u = 0; u < kFinCells / NW; ++u) {
        const int cl = warp + NW * u;
        const uint32_t s0 = __shfl_sync(0xFFFFFFFFu, f, cl);
        uint32_t s1 = cl < 31 ? __shfl_sync(0xFFFFFFFFu, f, cl + 1) : f_end;
        if (cl >= nc) s1 = s0;
        if (s1 == s0) continue;
        const float inv = mean ? 1.f / float(__ldg(cell_npts + c0 + cl)) : 1.f;
        for (uint32_t sg = s0; sg < s1; ++sg)
#pragma unroll
            for (int j = 0; j < CS; ++j)
                if (lane + 32 * j < C) rb[int64_t(sg) * C + 32 * j] = tile[lane + 32 * j][cl] * inv;
    }
}

struct TileBwdArgs {
    const float *grad_rows;  // (B, max_seg, C): tile_grad_rows_kernel's rows
    const void *feats;       // (B, N, C, H, W) f32; fused: the bf16 context
    const void *dist;        // (B, N, D, H, W) f32; fused: the bf16 depth logits
    const uint4 *hdr;
    const uint32_t *rec;
    const uint4 *groups;
    const uint32_t *seg_row;
    void *grad_feats;        // (B, N, C, H, W) f32 / bf16 (fused), or null
    void *grad_dist;         // (B, N, D, H, W) f32 / grad logits bf16 (fused), or null
    int64_t max_seg;
    TileGeom g;
    int C, wbudget;
};

// ---- tensor-core pieces of the backward (mma.sync m16n8k8, tf32 operands) ---
// fp32 accuracy from tf32 operands: x = hi + lo, hi = tf32(x), lo the exact
// fp32 remainder; a*b ~ hi*hi + hi*lo + lo*hi (the dropped lo*lo is 2^-22
// relative).  Measured 278 TFLOP/s for tf32 mma.sync on this GPU
// (scripts/mma_vs_ffma2.cu): the backward's two products per group -- the
// (row, segment) dot products over C channels and grad_f's 8-segment sums --
// are GEMM-shaped with K = C and N = C, where FFMA lanes-over-channels need a
// cross-lane reduction per dot product.
__device__ __forceinline__ void split_tf32(float x, uint32_t &hi, uint32_t &lo) {
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
    lo = __float_as_uint(x - __uint_as_float(hi));
}
// d += a * b three ways (lo*hi, hi*lo, hi*hi: small terms first)
__device__ __forceinline__ void mma3_tf32(float (&d)[4], const uint32_t (&ah)[4],
                                          const uint32_t (&al)[4], uint32_t bh0, uint32_t bh1,
                                          uint32_t bl0, uint32_t bl1) {
#define BVP_MMA_TF32(A, B0, B1)                                                        \
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, "       \
        "{%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"                                \
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])                               \
        : "r"(A[0]), "r"(A[1]), "r"(A[2]), "r"(A[3]), "r"(B0), "r"(B1))
    BVP_MMA_TF32(al, bh0, bh1);
    BVP_MMA_TF32(ah, bl0, bl1);
    BVP_MMA_TF32(ah, bh0, bh1);
#undef BVP_MMA_TF32
}

// One CTA per (tile, sample), clusters of CL columns as in the forward.  Per
// group (every warp every group; the group's 8 gradient rows copied to
// shared memory, double buffered):
//   Dot[h, k] = sum_c F[h, c] G[k, c]   -- M = 32 rows, N = 8 segments, K = C:
//     warp w takes m-tile w & 1 and k-steps w >> 1 (+4, +8) with its F
//     fragments held in registers; the 4 K-partials are added in a fixed
//     order through shared memory and written over the weight window's
//     (k, h) slots (A is read before);
//   grad_f[h, c] += sum_k A[k, h] G[k, c] -- M = 32 rows, N = C, K = 8:
//     warp w accumulates m-tile w & 1 x n-tiles w >> 1 (+4, +8) in registers
//     over all groups, in order.
// Then every point's record picks its Dot from the window into the
// depth-weight rows (weights no longer needed), points without a record
// are zeroed, grad_f goes over the feature rows, and both tiles go back to
// global memory through the cluster.  Deterministic (fixed sums, no atomics
// on values); tiles of <= 32 rows, C <= 128.
//
// FU (config F training, bvp_tile_fused_backward_bf16): the staging reads the
// bf16 context and depth logits and forms each pixel's depth softmax w in
// shared memory, as the fused forward does (its max and 1/sum kept per row);
// the records leave P = w grad_w in the weight rows, and each pixel row goes
// out as
//   grad_logit[d] = w[d] (grad_w[d] - sum_d' w[d'] grad_w[d'])
//                 = P[d] - w[d] sum_d' P[d']
// with w re-formed bit for bit from the (L2-resident) logits on the way out,
// so the shared footprint -- and 4 CTAs per SM -- is the fp32 variant's.
// Both gradients are rounded to bf16; no fp32 copy of the softmax, the
// context or a gradient touches global memory.
// FU's write-out of grad_logits (unstage_quads' item walk): for point
// (d, hl) of column j, P from column j's weight rows and the logit from
// global memory (read by the staging moments before: L2), then
//   w = exp2(l log2e - ms) inv  (the staging's arithmetic, the same bits)
//   grad_logit = P - w psum
template <int CL>
__device__ __forceinline__ void unstage_logit_grad(const ColumnXfer &x, __nv_bfloat16 *dst,
                                                   const __nv_bfloat16 *logits, int D,
                                                   int64_t base, const float *P, int stride,
                                                   const float *ms, const float *inv,
                                                   const float *psum) {
    constexpr int NW = kPoolThreads / 32, RS = 32 / CL, U = 4;
    constexpr float kLog2e = 1.4426950408889634f;
    const int warp = threadIdx.x >> 5;
    const int n_q = (((D + 3) >> 2) - x.rank + CL - 1) / CL;
    const int items = n_q * x.n_rb;
    for (int i0 = warp; i0 < items; i0 += NW * U) {
        int qs[U], mr[U];
        xfer_items<U>(i0, x.n_rb, qs, mr);
        float4 v[U];
        uint32_t l[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int it = i0 + NW * u;
            const int c0 = 4 * (x.rank + CL * qs[u]), hl = x.r0 + RS * mr[u];
            const bool ok = it < items && hl < x.th;
            v[u] = ok ? *reinterpret_cast<const float4 *>(P + hl * stride + c0)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
            const char *pl = reinterpret_cast<const char *>(
                logits + base + int64_t(c0) * x.HW + int64_t(hl) * x.W);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                l[u][e] = ldg_l2pf_u16(pl + 2 * int64_t(e) * x.HW, ok && c0 + e < D) << 16;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int it = i0 + NW * u;
            const int c0 = 4 * (x.rank + CL * qs[u]), hl = x.r0 + RS * mr[u];
            if (it < items && hl < x.th) {
                const float m = ms[hl], iv = inv[hl], s = psum[hl];
                __nv_bfloat16 *po = dst + base + int64_t(c0) * x.HW + int64_t(hl) * x.W;
                const float e4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (c0 + e < D) {
                        const float w = exp2f(fmaf(__uint_as_float(l[u][e]), kLog2e, -m)) * iv;
                        po[int64_t(e) * x.HW] = __float2bfloat16(e4[e] - w * s);
                    }
            }
        }
    }
}

// Register budget per variant, measured at S, B=4 (ncu): fp32 265 us at 4
// CTAs/SM (64 registers) against 289 at 3 (80); FU 336 at 4 against 323 at 3
// (its softmax, row sums and logit write-out keep more values live).
template <int CS, int CL, bool FU>
__global__ void __launch_bounds__(kPoolThreads, FU ? 3 : 4)
tile_backward_kernel(TileBwdArgs a) {
    constexpr int CP = CS * 32;
    constexpr int FS = CP + 4;   // = 4 (mod 32): conflict-free fragment loads
    constexpr int GS = CP + 4;
    extern __shared__ __align__(16) float sm[];
    __shared__ uint32_t s_cov[kTileMaxPoints / 32];  // points with a record
    __shared__ float s_dpart[4][32][kTileGroup];      // Dot K-partials of a group
    __shared__ float s_a[32][kTileGroup + 1];          // the group's A, dense [row][segment]
    const TileGeom &g = a.g;
    const int64_t t = blockIdx.x;
    const int b = blockIdx.y;
    const TileId id = tile_id(t, g.W, g.n_hb, g.TH, g.H);
    const uint4 h = a.hdr[t];
    const int n_segs = int(h.y), n_groups = int(h.z);
    const int HW = g.H * g.W, C = a.C, D = g.D, PD = (D + 3) & ~3;
    float *ws = sm;               // weight window [wbudget]: A, then the dot products
    float *fs = ws + a.wbudget;   // [TH][FS] feature rows, then grad_f rows
    float *pw = fs + g.TH * FS;   // [TH][PD] depth weights, then grad_w rows
    float *gsm = pw + g.TH * PD;  // [2][8][GS] gradient rows of the current / next group
    __shared__ float s_ms[FU ? 32 : 1], s_inv[FU ? 32 : 1], s_psum[FU ? 32 : 1];  // FU, per row
    const int64_t nb = int64_t(b) * g.N + id.n;
    const int64_t pix0 = int64_t(id.h0) * g.W + id.w;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g8 = lane >> 2, t4 = lane & 3;
    const int mt = warp & 1, wq4 = warp >> 1;  // m-tile; k-step / n-tile quarter
    const int NT = (C + 7) >> 3;               // n-tiles (and k-steps) over C
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = CL > 1 ? int(cluster.block_rank()) : 0;
    const ColumnXfer x = column_xfer<CL>(rank, id.th, HW, g.W);
    const int64_t col = pix0 - rank + x.j;
    if (CL > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    for (int i = threadIdx.x; i < kTileMaxPoints / 32; i += kPoolThreads) s_cov[i] = 0u;
    // gradient-row buffers: channels past C stay zero (the copies stop at C)
    for (int i = threadIdx.x; i < 2 * kTileGroup * GS; i += kPoolThreads) gsm[i] = 0.f;
    // the first weight window's zeros (windows are multiples of 8 floats)
    for (uint32_t i = 4 * threadIdx.x; i < min(h.w, uint32_t(a.wbudget)); i += 4 * kPoolThreads)
        *reinterpret_cast<float4 *>(ws + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    {
        float *rfs = CL > 1 ? cluster.map_shared_rank(fs, x.j) : fs;
        float *rpw = CL > 1 ? cluster.map_shared_rank(pw, x.j) : pw;
        constexpr int ES = FU ? 2 : 4;
        stage_quads<CL, ES>(x, a.feats, C, CP / 4, nb * C * HW + col, rfs, FS, true);
        stage_quads<CL, ES>(x, a.dist, D, (D + 3) >> 2, nb * D * HW + col, rpw, PD, false);
        if (CL > 1) cluster.sync();
        else __syncthreads();
    }
    if (FU) {
        // w = softmax_D of each pixel row in place (lift.py:17-31, fp32 from
        // bf16 logits), 8 lanes per pixel as in the fused forward; the
        // aggregation below reads it after its barrier
        constexpr float kLog2e = 1.4426950408889634f;
        const int sub = lane & 7;
        for (int hl0 = 4 * warp; hl0 < id.th; hl0 += 4 * (kPoolThreads / 32)) {
            const int hl = hl0 + (lane >> 3);
            const bool on = hl < id.th;
            float *row = pw + (on ? hl : 0) * PD;
            float m = -INFINITY;
            if (on)
                for (int d = sub; d < D; d += 8) m = fmaxf(m, row[d]);
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
            const float ms = m * kLog2e;
            float sum = 0.f;
            if (on)
                for (int d = sub; d < D; d += 8) {
                    const float e = exp2f(fmaf(row[d], kLog2e, -ms));
                    row[d] = e;
                    sum += e;
                }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
            const float inv = 1.f / sum;
            if (on)
                for (int d = sub; d < D; d += 8) row[d] *= inv;
            if (on && sub == 0) {
                s_ms[hl] = ms;
                s_inv[hl] = inv;
            }
        }
    }
    // this warp's F fragments (A operand of Dot): rows mt*16 + g (+8),
    // channels 8 ks + t (+4), k-steps ks = wq4, wq4 + 4, wq4 + 8
    uint32_t fh[3][4], fl[3][4];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int ks = wq4 + 4 * i;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int r = mt * 16 + g8 + 8 * (e & 1), c = 8 * ks + t4 + 4 * (e >> 1);
            const float v = ks < NT && r < id.th ? fs[r * FS + c] : 0.f;
            split_tf32(v, fh[i][e], fl[i][e]);
        }
    }
    float gacc[3][4];  // grad_f: m-tile mt x n-tiles wq4 (+4, +8)
#pragma unroll
    for (int i = 0; i < 3; ++i) gacc[i][0] = gacc[i][1] = gacc[i][2] = gacc[i][3] = 0.f;
    const uint4 *gt = a.groups + t * g.gcap;
    const uint32_t *srow = a.seg_row + t * g.tpc;
    const uint32_t *rt = a.rec + t * g.tpc;
    const float *grows0 = a.grad_rows + int64_t(b) * a.max_seg * C;
    const int shift = g.hl_bits + g.d_bits;
    const uint32_t dmask = (1u << g.d_bits) - 1u, hmask = (1u << g.hl_bits) - 1u;
    const uint32_t wmask = (1u << (30 - shift)) - 1u;
    const uint32_t total_w = h.w;
    // the copy's 16-byte item of this thread (8 x C/4 <= 256 items: at most one)
    const int f_c4 = C >> 2, f_k = threadIdx.x / max(f_c4, 1);
    const int f_c = 4 * (threadIdx.x - f_k * f_c4);
    auto fetch = [&](int q, int buf) {  // group q's gradient rows -> gsm[buf]
        const int nk = min(kTileGroup, n_segs - q * kTileGroup);
        float *dst = gsm + buf * (kTileGroup * GS);
        if ((C & 3) == 0) {
            if (f_k < kTileGroup) {
                const int k = f_k, c = f_c;
                if (k < nk) {
                    const float *src = grows0 + int64_t(srow[q * kTileGroup + k]) * C + c;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     static_cast<uint32_t>(__cvta_generic_to_shared(dst + k * GS + c))),
                                 "l"(src));
                } else {  // rows past the group's cells: zero (their A is 0)
                    *reinterpret_cast<float4 *>(dst + k * GS + c) = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        } else {
            for (int i = threadIdx.x; i < kTileGroup * C; i += kPoolThreads) {
                const int k = i / C, c = i - k * C;
                if (k < nk) {
                    const float *src = grows0 + int64_t(srow[q * kTileGroup + k]) * C + c;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                     static_cast<uint32_t>(__cvta_generic_to_shared(dst + k * GS + c))),
                                 "l"(src));
                } else {
                    dst[k * GS + c] = 0.f;
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int q0 = 0; q0 < n_groups;) {
        // weight windows as in the forward (one for nearly every tile)
        const uint4 G0 = q0 ? gt[q0] : make_uint4(0u, 0u, 0u, 0u);
        int q1 = n_groups;
        if (total_w - G0.z > uint32_t(a.wbudget)) {
            int lo = q0 + 1, hi = n_groups - 1;
            q1 = q0 + 1;
            while (lo <= hi) {
                const int mid = (lo + hi) >> 1;
                if (gt[mid].z - G0.z <= uint32_t(a.wbudget)) {
                    q1 = mid;
                    lo = mid + 1;
                } else {
                    hi = mid - 1;
                }
            }
        }
        const uint32_t r_end = q1 == n_groups ? h.x : gt[q1].w;
        const uint32_t w_end = q1 == n_groups ? total_w : gt[q1].z;
        if (q0 > 0) {  // (the first window was zeroed beside the staging)
            __syncthreads();  // previous window's records done with ws / pw
            for (uint32_t i = 4 * threadIdx.x; i < w_end - G0.z; i += 4 * kPoolThreads)
                *reinterpret_cast<float4 *>(ws + i) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        fetch(q0, 0);
        __syncthreads();
        // aggregation: A of the window (the forward's arithmetic); each
        // thread's records 8 at a time, all loaded before any is used
        for (uint32_t k0 = G0.w + threadIdx.x; k0 < r_end; k0 += 8 * kPoolThreads) {
            uint32_t rr[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t k = k0 + u * kPoolThreads;
                rr[u] = k < r_end ? __ldg(rt + k) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                uint32_t r = rr[u];
                if (!(r >> 31)) continue;
                const uint32_t widx = (r >> shift) & wmask;
                float sum = pw[((r >> g.d_bits) & hmask) * PD + (r & dmask)];
                for (uint32_t kk = k0 + u * kPoolThreads + 1; (r >> 30) & 1u; ++kk) {
                    r = __ldg(rt + kk);
                    sum += pw[((r >> g.d_bits) & hmask) * PD + (r & dmask)];
                }
                ws[widx - G0.z] = sum;
            }
        }
        // this thread's (row, segment) of a group: its window slot; the
        // group's A goes dense into s_a for the fragments
        const int ar = threadIdx.x >> 3, ak = threadIdx.x & 7;
        int a_slot = 0;
        bool a_in = false;
        auto load_a = [&](int q) {
            const uint4 Gq = gt[q];
            const unsigned long long m = Gq.x | (static_cast<unsigned long long>(Gq.y) << 32);
            const int nk = min(kTileGroup, n_segs - q * kTileGroup);
            a_in = ak < nk && ar < id.th && ((m >> ar) & 1ull);
            a_slot = (Gq.z - G0.z) + (a_in ? __popcll(m & ((1ull << ar) - 1ull)) * kTileGroup + ak : 0);
            s_a[ar][ak] = a_in ? ws[a_slot] : 0.f;
        };
        __syncthreads();  // A of the window complete
        load_a(q0);
        for (int q = q0; q < q1; ++q) {
            if (q + 1 < q1) {
                fetch(q + 1, (q + 1 - q0) & 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();  // group q's rows and s_a visible; s_dpart free
            const float *gq = gsm + ((q - q0) & 1) * (kTileGroup * GS);
            // Dot K-partial: this warp's k-steps
            {
                float dacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const int ks = wq4 + 4 * i;
                    if (ks < NT) {  // B = G^T: b0 = G[g][8 ks + t], b1 = G[g][8 ks + t + 4]
                        uint32_t bh0, bl0, bh1, bl1;
                        split_tf32(gq[g8 * GS + 8 * ks + t4], bh0, bl0);
                        split_tf32(gq[g8 * GS + 8 * ks + t4 + 4], bh1, bl1);
                        mma3_tf32(dacc, fh[i], fl[i], bh0, bh1, bl0, bl1);
                    }
                }
                // rows mt*16 + g (+8), segments 2t, 2t+1
                s_dpart[wq4][mt * 16 + g8][2 * t4] = dacc[0];
                s_dpart[wq4][mt * 16 + g8][2 * t4 + 1] = dacc[1];
                s_dpart[wq4][mt * 16 + g8 + 8][2 * t4] = dacc[2];
                s_dpart[wq4][mt * 16 + g8 + 8][2 * t4 + 1] = dacc[3];
            }
            // grad_f: A^T (rows x segments) . G (segments x channels)
            {
                const int r0 = mt * 16 + g8;
                const float a4[4] = {s_a[r0][t4], s_a[r0 + 8][t4], s_a[r0][t4 + 4],
                                     s_a[r0 + 8][t4 + 4]};
                uint32_t ah[4], al[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) split_tf32(a4[e], ah[e], al[e]);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const int nt = wq4 + 4 * i;
                    if (nt < NT) {  // b0 = G[t][8 nt + g], b1 = G[t + 4][8 nt + g]
                        uint32_t bh0, bl0, bh1, bl1;
                        split_tf32(gq[t4 * GS + 8 * nt + g8], bh0, bl0);
                        split_tf32(gq[(t4 + 4) * GS + 8 * nt + g8], bh1, bl1);
                        mma3_tf32(gacc[i], ah, al, bh0, bh1, bl0, bl1);
                    }
                }
            }
            __syncthreads();  // partials complete; every warp done with s_a and this buffer
            // Dot = the 4 K-partials in order, over the window's (k, h) slots;
            // then the next group's A
            if (a_in)
                ws[a_slot] = ((s_dpart[0][ar][ak] + s_dpart[1][ar][ak]) + s_dpart[2][ar][ak]) +
                             s_dpart[3][ar][ak];
            if (q + 1 < q1) load_a(q + 1);
        }
        __syncthreads();
        // every point of the window: its Dot into the depth-weight rows (the
        // records 8 at a time, as above)
        for (uint32_t k0 = G0.w + threadIdx.x; k0 < r_end; k0 += 8 * kPoolThreads) {
            uint32_t rr[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t k = k0 + u * kPoolThreads;
                rr[u] = k < r_end ? __ldg(rt + k) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (k0 + u * kPoolThreads >= r_end) break;
                const uint32_t r = rr[u];
                const uint32_t hl = (r >> g.d_bits) & hmask, d = r & dmask;
                const float dot = ws[((r >> shift) & wmask) - G0.z];
                if (FU) pw[hl * PD + d] *= dot;  // P = w grad_w
                else pw[hl * PD + d] = dot;
                const uint32_t pt = hl * uint32_t(D) + d;
                atomicOr(&s_cov[pt >> 5], 1u << (pt & 31));
            }
        }
        q0 = q1;
    }
    __syncthreads();
    // points without a record (out of range) get a zero weight gradient; the
    // grad_f fragments go over the feature rows
    for (int hl = warp; hl < id.th; hl += kPoolThreads / 32) {
        if (!FU) {
            for (int d = lane; d < D; d += 32) {
                const int pt = hl * D + d;
                if (!((s_cov[pt >> 5] >> (pt & 31)) & 1u)) pw[hl * PD + d] = 0.f;
            }
            continue;
        }
        // FU: P of points without a record is 0; the row's sum of P (lane
        // partials, then a fixed butterfly: deterministic)
        float *pr = pw + hl * PD;
        float s = 0.f;
        for (int d = lane; d < D; d += 32) {
            const int pt = hl * D + d;
            if ((s_cov[pt >> 5] >> (pt & 31)) & 1u) s += pr[d];
            else pr[d] = 0.f;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
        if (lane == 0) s_psum[hl] = s;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int nt = wq4 + 4 * i;
        if (nt >= NT) continue;
        const int r0 = mt * 16 + g8, c0 = 8 * nt + 2 * t4;
        if (r0 < id.th) {
            fs[r0 * FS + c0] = gacc[i][0];
            fs[r0 * FS + c0 + 1] = gacc[i][1];
        }
        if (r0 + 8 < id.th) {
            fs[(r0 + 8) * FS + c0] = gacc[i][2];
            fs[(r0 + 8) * FS + c0 + 1] = gacc[i][3];
        }
    }
    if (CL > 1) cluster.sync();
    else __syncthreads();
    {
        using OT = typename std::conditional<FU, __nv_bfloat16, float>::type;
        const float *rfs = CL > 1 ? cluster.map_shared_rank(fs, x.j) : fs;
        const float *rpw = CL > 1 ? cluster.map_shared_rank(pw, x.j) : pw;
        if (a.grad_feats)
            unstage_quads<CL>(x, static_cast<OT *>(a.grad_feats), C, nb * C * HW + col, rfs, FS);
        if (a.grad_dist) {
            if (FU) {
                const float *rms = CL > 1 ? cluster.map_shared_rank(s_ms, x.j) : s_ms;
                const float *rinv = CL > 1 ? cluster.map_shared_rank(s_inv, x.j) : s_inv;
                const float *rps = CL > 1 ? cluster.map_shared_rank(s_psum, x.j) : s_psum;
                unstage_logit_grad<CL>(x, static_cast<__nv_bfloat16 *>(a.grad_dist),
                                       static_cast<const __nv_bfloat16 *>(a.dist), D,
                                       nb * D * HW + col, rpw, PD, rms, rinv, rps);
            } else {
                unstage_quads<CL>(x, static_cast<float *>(a.grad_dist), D, nb * D * HW + col,
                                  rpw, PD);
            }
        }
    }
    if (CL > 1) cluster.sync();  // peers done reading this CTA's shared memory
}

template <int CS, int CL, bool FU>
static int launch_backward(const TileBwdArgs &a, int B, size_t smem, cudaStream_t s) {
    static int max_dyn = -1;
    if (max_dyn < 0) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, tile_backward_kernel<CS, CL, FU>);
        max_dyn = 227 * 1024 - int(fa.sharedSizeBytes);
        cudaFuncSetAttribute(tile_backward_kernel<CS, CL, FU>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
    }
    BVP_REQUIRE(smem <= size_t(max_dyn), BVP_ERR_UNSUPPORTED,
                "tile backward needs %zu bytes of shared memory (max %d)", smem, max_dyn);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(a.g.T), unsigned(B));
    cfg.blockDim = dim3(kPoolThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr_c[1];
    attr_c[0].id = cudaLaunchAttributeClusterDimension;
    attr_c[0].val.clusterDim.x = CL;
    attr_c[0].val.clusterDim.y = 1;
    attr_c[0].val.clusterDim.z = 1;
    cfg.attrs = attr_c;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, tile_backward_kernel<CS, CL, FU>, a);
    BVP_REQUIRE(e == cudaSuccess, BVP_ERR_CUDA, "tile_backward launch: %s", cudaGetErrorString(e));
    return BVP_OK;
}

template <int CS, bool FU>
static int run_tile_backward(const float *grad_out, const void *feats, const void *dist,
                             const bvp_tile_plan *p, const TileGeom &g, int B, int C, int mean,
                             float *rows, void *grad_feats, void *grad_dist, cudaStream_t s) {
    const PlanLayout L = plan_layout(g, p->n_cells);
    tile_grad_rows_kernel<CS><<<dim3(unsigned(ceil_div(p->n_cells, kFinCells)), unsigned(B)),
                                kPoolThreads, 0, s>>>(
        grad_out, at<const uint32_t>(p, L.csf), at<const uint32_t>(p, L.npts), int(p->n_cells), C,
        mean, p->max_seg, rows);
    TileBwdArgs a{};
    a.grad_rows = rows;
    a.feats = feats;
    a.dist = dist;
    a.hdr = at<const uint4>(p, L.hdr);
    a.rec = at<const uint32_t>(p, L.rec);
    a.groups = at<const uint4>(p, L.groups);
    a.seg_row = at<const uint32_t>(p, L.seg_row);
    a.grad_feats = grad_feats;
    a.grad_dist = grad_dist;
    a.max_seg = p->max_seg;
    a.g = g;
    a.C = C;
    a.wbudget = std::max(2048, 128 * g.TH);
    const int CP = CS * 32;
    const size_t smem = sizeof(float) * (size_t(g.TH) * (CP + 4) + size_t(g.TH) * ((g.D + 3) & ~3) +
                                         a.wbudget + 2 * kTileGroup * (CP + 4));
    const int CL = (g.W % 8 == 0) ? 8 : (g.W % 4 == 0) ? 4 : (g.W % 2 == 0) ? 2 : 1;
    int rc;
    switch (CL) {
        case 8: rc = launch_backward<CS, 8, FU>(a, B, smem, s); break;
        case 4: rc = launch_backward<CS, 4, FU>(a, B, smem, s); break;
        case 2: rc = launch_backward<CS, 2, FU>(a, B, smem, s); break;
        default: rc = launch_backward<CS, 1, FU>(a, B, smem, s); break;
    }
    if (rc != BVP_OK) return rc;
    return check_launch(FU ? "tile_fused_backward" : "tile_backward");
}

template <bool FU>
static int tile_backward_dispatch(const float *grad_out, const void *feats, const void *dist,
                                  const bvp_tile_plan *plan, int B, int C, int mode, float *rows,
                                  size_t rows_bytes, void *grad_feats, void *grad_dist,
                                  void *stream) {
    TileGeom g;
    const int rc = plan_dims_from(plan, g);
    if (rc != BVP_OK) return rc;
    BVP_REQUIRE(B >= 1 && C >= 0, BVP_ERR_INVALID, "bad dims B=%d C=%d", B, C);
    BVP_REQUIRE(mode == BVP_SUM || mode == BVP_MEAN, BVP_ERR_UNSUPPORTED,
                "the tiled backward takes SUM and MEAN only (mode %d)", mode);
    BVP_REQUIRE(C <= 128, BVP_ERR_UNSUPPORTED, "the tiled backward takes C <= 128 (C=%d)", C);
    BVP_REQUIRE(g.TH <= 32, BVP_ERR_UNSUPPORTED, "the tiled backward takes tiles of <= 32 rows");
    if (!grad_feats && !grad_dist) return BVP_OK;
    if (C == 0) {  // no channels: the weights' gradient is zero (grad_features is empty)
        if (grad_dist)
            cudaMemsetAsync(grad_dist, 0,
                            size_t(B) * g.N * g.D * g.H * g.W * (FU ? 2 : sizeof(float)),
                            as_stream(stream));
        return check_launch(FU ? "tile_fused_backward" : "tile_backward");
    }
    BVP_REQUIRE(grad_out && feats && dist && rows, BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(rows_bytes >= size_t(B) * plan->max_seg * C * sizeof(float), BVP_ERR_INVALID,
                "segment-row scratch too small: need %zu bytes, got %zu",
                size_t(B) * plan->max_seg * C * sizeof(float), rows_bytes);
    cudaStream_t s = as_stream(stream);
    const int mean = mode == BVP_MEAN;
    switch ((C + 31) / 32) {
        case 1: return run_tile_backward<1, FU>(grad_out, feats, dist, plan, g, B, C, mean, rows,
                                                grad_feats, grad_dist, s);
        case 2: return run_tile_backward<2, FU>(grad_out, feats, dist, plan, g, B, C, mean, rows,
                                                grad_feats, grad_dist, s);
        case 3: return run_tile_backward<3, FU>(grad_out, feats, dist, plan, g, B, C, mean, rows,
                                                grad_feats, grad_dist, s);
        default: return run_tile_backward<4, FU>(grad_out, feats, dist, plan, g, B, C, mean, rows,
                                                 grad_feats, grad_dist, s);
    }
}

}  // namespace bvp

using namespace bvp;

extern "C" {

int bvp_tile_backward_f32(const float *grad_out, const float *features, const float *dist,
                          const bvp_tile_plan *plan, int B, int C, int mode, float *rows,
                          size_t rows_bytes, float *grad_features, float *grad_dist,
                          void *stream) {
    return tile_backward_dispatch<false>(grad_out, features, dist, plan, B, C, mode, rows,
                                         rows_bytes, grad_features, grad_dist, stream);
}

int bvp_tile_fused_backward_bf16(const float *grad_out, const uint16_t *logits,
                                 const uint16_t *context, const bvp_tile_plan *plan, int B, int C,
                                 int mode, float *rows, size_t rows_bytes, uint16_t *grad_logits,
                                 uint16_t *grad_context, void *stream) {
    return tile_backward_dispatch<true>(grad_out, context, logits, plan, B, C, mode, rows,
                                        rows_bytes, grad_context, grad_logits, stream);
}

}  // extern "C"

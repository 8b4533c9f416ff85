// tile.cu -- pixel-column tiled BEV pooling (SUM / MEAN, fp32 accumulate).
//
// The reference reduces interval by interval: every in-range point of a
// cell gathers its pixel's feature row (_kernels.py:34-55).  A pixel's row is
// used by every depth bin of its ray (~103 points at the nuScenes shape), so
// the interval formulation re-reads each 320-byte row ~100 times from L2.
// Here the work is tiled by PIXELS instead of by cells:
//
//   tile t = one camera column segment (n, w, rows h0..h0+TH): its TH feature
//   rows are staged in shared memory ONCE; every point of the tile is one
//   (h, d) of those rows.  Within the tile the points are sorted by cell
//   (then h, d); a run of equal cells is a "segment".  8 consecutive
//   segments form a group, and a group is a small dense product
//
//       seg_row[k, c] = sum_{h in union(g)} A[k, h] * F[h, c],   k < 8
//       A[k, h]       = sum_{d : cell(h, d) = cell_k} w[h, d]
//
//   (the union is the set of rows any of the 8 cells sees; for a level rig
//   all rows of a column hit the same cells, so A is ~97% dense at S).
//   One warp computes a group with lanes over channels, 8 x ceil(C/32)
//   accumulators per lane, the row of F read once per (group, h) for all 8
//   cells.
//
// Phase 1 (tile_pool_kernel, one CTA per (tile, sample)) writes one 4C-byte
// row per segment; phase 2 (tile_finalize_kernel, one CTA per 32 cells)
// sums each cell's segment rows in tile order (~22% of cells at S see more
// than one tile), applies MEAN's 1/len, transposes through shared memory and
// writes the channel-major map (C, n_cells) with full 128-byte lines -- every
// element exactly once, empty cells as zeros (pooling.py:213).  No atomics
// touch values: the result is deterministic and independent of launch shape.
//
// The plan (tile_plan_kernel and friends) is built once per association on
// the GPU: from the association's ranks by a stable partition by tile
// (bvp_build_tile_plan_ranks), or from cell_of_point alone (bevgrid.py:85-98's
// output) by a per-tile sort (bvp_build_tile_plan); the two plans are equal.
// The adjoint is tile_backward.cu; shared pieces are in tile.cuh.
//
// Reference: pooling.py:206-221 (pool_interval), _kernels.py:22-63
// (interval_reduce), bevgrid.py:142-158 (the association it consumes).
#include "tile.cuh"

namespace bvp {

// ---- plan build -------------------------------------------------------------
// Tile of a frustum point id p = ((n H + h) W + w) D + d.
__device__ __forceinline__ uint32_t tile_of_point(uint32_t p, const TileGeom &g) {
    const uint32_t pix = p / uint32_t(g.D);
    const uint32_t w = pix % uint32_t(g.W), nh = pix / uint32_t(g.W);
    const uint32_t h = nh % uint32_t(g.H), n = nh / uint32_t(g.H);
    return (n * uint32_t(g.n_hb) + h / uint32_t(g.TH)) * uint32_t(g.W) + w;
}

// The association's ranks (in-range point ids, by cell, ties by id) keyed by
// their tile, and the points per tile (block histogram in shared memory,
// one global add per tile and block).  A stable partition of the ranks by
// these keys lists every tile's points by (cell, h, d): the tile's own order.
__global__ void tile_key_kernel(const uint32_t *__restrict__ ranks,
                                const int64_t *__restrict__ counts, TileGeom g, int64_t P,
                                uint32_t *__restrict__ keys, uint32_t *__restrict__ tile_count) {
    extern __shared__ uint32_t s_hist[];  // [T]
    const uint32_t T = uint32_t(g.T);
    for (uint32_t i = threadIdx.x; i < T; i += blockDim.x) s_hist[i] = 0u;
    __syncthreads();
    const int64_t n_in = counts[0];
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < P;
         j += int64_t(gridDim.x) * blockDim.x) {
        uint32_t k = kOOR;
        if (j < n_in) {
            k = tile_of_point(__ldg(ranks + j), g);
            atomicAdd(&s_hist[k], 1u);
        }
        keys[j] = k;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < T; i += blockDim.x)
        if (s_hist[i]) atomicAdd(tile_count + i, s_hist[i]);
}

// The tile's points from the association, in order (SORTED plan build):
// pts[start[t], start[t + 1]) are tile t's point ids by (cell, h, d).
struct TileSorted {
    const uint32_t *pts;
    const uint32_t *start;
};

// One CTA per tile.  Keys (cell << 16 | hl << d_bits | d), ascending; the
// low bits order the points of a cell by (h, d), which is their rank order
// within the tile (bevgrid.py:149's stable tie-break restricted to one
// column).  SORTED: read in that order from the association (TileSorted);
// otherwise sorted in shared memory (bitonic) from cell_of_point alone.
template <bool SORTED>
__global__ void __launch_bounds__(kPlanThreads)
tile_plan_kernel(const uint32_t *__restrict__ cells, TileGeom g, uint4 *__restrict__ hdr,
                 uint32_t *__restrict__ rec, uint32_t *__restrict__ seg_cell,
                 uint32_t *__restrict__ seg_start, uint4 *__restrict__ groups,
                 int *__restrict__ err, TileSorted ts) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long *keys = reinterpret_cast<unsigned long long *>(smem);
    __shared__ unsigned long long gmask[kTileMaxPoints / kTileGroup + 1];
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_tot[2];

    const int64_t t = blockIdx.x;
    const TileId id = tile_id(t, g.W, g.n_hb, g.TH, g.H);
    const int np_all = id.th * g.D;
    int cap = 1;
    while (cap < np_all) cap <<= 1;
    const uint32_t *cbase = cells + ((int64_t(id.n) * g.H + id.h0) * g.W + id.w) * g.D;
    const int64_t hstride = int64_t(g.W) * g.D;
    uint32_t nvalid = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int i = threadIdx.x; i < kTileMaxPoints / kTileGroup + 1; i += blockDim.x) gmask[i] = 0;
    const int hmask = (1 << g.hl_bits) - 1, dmask = (1 << g.d_bits) - 1;
    int n_pts;
    if (SORTED) {
        const uint32_t lo = __ldg(ts.start + t), hi = __ldg(ts.start + t + 1);
        n_pts = int(hi - lo);
        for (int k = threadIdx.x; k < n_pts; k += blockDim.x) {
            const uint32_t p = __ldg(ts.pts + lo + k);
            const uint32_t pix = p / uint32_t(g.D), d = p - pix * uint32_t(g.D);
            const uint32_t hl = (pix / uint32_t(g.W)) % uint32_t(g.H) - uint32_t(id.h0);
            keys[k] = (static_cast<unsigned long long>(__ldg(cells + p)) << 16) |
                      ((hl << g.d_bits) | d);
        }
        __syncthreads();
    } else {
        for (int hl = warp; hl < id.th; hl += nw)
            for (int d = lane; d < g.D; d += 32) {
                const uint32_t c = __ldg(cbase + hl * hstride + d);
                unsigned long long k = ~0ull;
                if (c != kOOR) {
                    k = (static_cast<unsigned long long>(c) << 16) |
                        static_cast<unsigned>((hl << g.d_bits) | d);
                    ++nvalid;
                }
                keys[hl * g.D + d] = k;
            }
        for (int i = np_all + threadIdx.x; i < cap; i += blockDim.x) keys[i] = ~0ull;
        block_excl_scan(nvalid, s_warp, &s_tot[0]);
        n_pts = int(s_tot[0]);
    }
    // bitonic sort of keys[0, cap)
    if (!SORTED) {
        for (int k = 2; k <= cap; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < (cap >> 1); i += blockDim.x) {
                    const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;
                    const unsigned long long a = keys[lo], b = keys[hi];
                    const bool up = (lo & k) == 0;
                    if ((a > b) == up) {
                        keys[lo] = b;
                        keys[hi] = a;
                    }
                }
                __syncthreads();
            }
        }
    }
    // segments: thread owns the contiguous points [k0, k1)
    const int per = (n_pts + blockDim.x - 1) / blockDim.x;
    const int k0 = min(n_pts, int(threadIdx.x) * per), k1 = min(n_pts, k0 + per);
    uint32_t heads = 0;
    for (int k = k0; k < k1; ++k)
        heads += (k == 0 || (keys[k] >> 16) != (keys[k - 1] >> 16)) ? 1u : 0u;
    uint32_t seg = block_excl_scan(heads, s_warp, &s_tot[1]);
    const int n_segs = int(s_tot[1]);
    const int n_groups = (n_segs + kTileGroup - 1) / kTileGroup;
    // union masks of the groups
    {
        uint32_t sg = seg;
        for (int k = k0; k < k1; ++k) {
            const bool head = (k == 0 || (keys[k] >> 16) != (keys[k - 1] >> 16));
            if (head) ++sg;
            const int hl = int(keys[k] >> g.d_bits) & hmask;
            atomicOr(&gmask[(sg - 1) / kTileGroup], 1ull << hl);
        }
    }
    __syncthreads();
    // group offsets into the weight window: 8 floats per union row
    __shared__ uint32_t s_woff[kTileMaxPoints / kTileGroup + 1];
    {
        const int gper = (n_groups + blockDim.x - 1) / blockDim.x;
        const int g0 = min(n_groups, int(threadIdx.x) * gper), g1 = min(n_groups, g0 + gper);
        uint32_t sum = 0;
        for (int q = g0; q < g1; ++q) sum += kTileGroup * __popcll(gmask[q]);
        uint32_t off = block_excl_scan(sum, s_warp, &s_tot[0]);
        for (int q = g0; q < g1; ++q) {
            s_woff[q] = off;
            off += kTileGroup * __popcll(gmask[q]);
        }
    }
    __syncthreads();
    const uint32_t total_w = s_tot[0];
    const int shift = g.hl_bits + g.d_bits;
    const uint32_t wmax = 1u << (30 - shift);
    if (threadIdx.x == 0 && total_w > wmax) atomicExch(err, 1);
    uint4 *gt = groups + t * g.gcap;
    uint32_t *rt = rec + t * g.tpc;
    uint32_t *sc = seg_cell + t * g.tpc;
    uint32_t *sn = seg_start + t * g.tpc;
    {
        uint32_t sg = seg;  // segments started before k0
        for (int k = k0; k < k1; ++k) {
            const uint32_t c = uint32_t(keys[k] >> 16);
            const bool head = (k == 0 || c != uint32_t(keys[k - 1] >> 16));
            if (head) ++sg;
            const uint32_t s = sg - 1;
            const int hl = int(keys[k] >> g.d_bits) & hmask, d = int(keys[k]) & dmask;
            const int q = int(s / kTileGroup), kk = int(s % kTileGroup);
            const int prev_hl = k > 0 ? int(keys[k - 1] >> g.d_bits) & hmask : -1;
            const bool run_head = head || hl != prev_hl;
            const unsigned long long m = gmask[q];
            const uint32_t upos = __popcll(m & ((1ull << hl) - 1ull));
            const uint32_t widx = s_woff[q] + upos * kTileGroup + kk;
            // bit 31: first point of a (cell, row) run; bit 30: the run goes on
            // with the next record (most runs are single points: their
            // aggregation then reads no other record)
            const bool more = k + 1 < n_pts && uint32_t(keys[k + 1] >> 16) == c &&
                              (int(keys[k + 1] >> g.d_bits) & hmask) == hl;
            rt[k] = (run_head ? 0x80000000u : 0u) | (more ? 0x40000000u : 0u) |
                    ((widx & (wmax - 1)) << shift) | (uint32_t(hl) << g.d_bits) | uint32_t(d);
            if (head) {
                sc[s] = c;
                sn[s] = uint32_t(k);  // first point of the segment
                if (kk == 0)
                    gt[q] = make_uint4(uint32_t(m), uint32_t(m >> 32), s_woff[q], uint32_t(k));
            }
        }
    }
    if (threadIdx.x == 0) {
        gt[n_groups] = make_uint4(0u, 0u, total_w, uint32_t(n_pts));
        hdr[t] = make_uint4(uint32_t(n_pts), uint32_t(n_segs), uint32_t(n_groups), total_w);
    }
}

// Segments per cell (and in-range points per cell, for MEAN).
__global__ void tile_seg_count_kernel(const uint4 *__restrict__ hdr, TileGeom g,
                                      const uint32_t *__restrict__ seg_cell,
                                      const uint32_t *__restrict__ seg_start,
                                      uint32_t *__restrict__ cell_nseg,
                                      uint32_t *__restrict__ cell_npts) {
    const int64_t t = blockIdx.x;
    const int n_segs = int(hdr[t].y);
    for (int s = threadIdx.x; s < n_segs; s += blockDim.x) {
        const uint32_t c = seg_cell[t * g.tpc + s];
        const uint32_t first = seg_start[t * g.tpc + s];
        const uint32_t end = s + 1 < n_segs ? seg_start[t * g.tpc + s + 1] : hdr[t].x;
        atomicAdd(&cell_nseg[c], 1u);
        atomicAdd(&cell_npts[c], end - first);
    }
}

// Slots in arrival order; tile_seg_fix_kernel reorders them by tile.
__global__ void tile_seg_assign_kernel(const uint4 *__restrict__ hdr, TileGeom g,
                                       const uint32_t *__restrict__ seg_cell,
                                       const uint32_t *__restrict__ cell_seg_first,
                                       uint32_t *__restrict__ cell_fill,
                                       unsigned long long *__restrict__ owner) {
    const int64_t t = blockIdx.x;
    const int n_segs = int(hdr[t].y);
    for (int s = threadIdx.x; s < n_segs; s += blockDim.x) {
        const uint32_t c = seg_cell[t * g.tpc + s];
        const uint32_t slot = atomicAdd(&cell_fill[c], 1u);
        owner[cell_seg_first[c] + slot] = (static_cast<unsigned long long>(t) << 32) | uint32_t(s);
    }
}

// Per cell: order its segments by tile (deterministic), record each
// segment's row index.
__global__ void tile_seg_fix_kernel(const uint32_t *__restrict__ cell_seg_first, int64_t n_cells,
                                    TileGeom g, unsigned long long *__restrict__ owner,
                                    uint32_t *__restrict__ seg_row) {
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_cells;
         c += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t s0 = cell_seg_first[c], s1 = cell_seg_first[c + 1];
        if (s1 - s0 > 1) {  // insertion sort (a few entries)
            for (uint32_t a = s0 + 1; a < s1; ++a) {
                const unsigned long long v = owner[a];
                uint32_t b = a;
                while (b > s0 && owner[b - 1] > v) {
                    owner[b] = owner[b - 1];
                    --b;
                }
                owner[b] = v;
            }
        }
        for (uint32_t a = s0; a < s1; ++a) {
            const unsigned long long v = owner[a];
            seg_row[int64_t(v >> 32) * g.tpc + uint32_t(v)] = a;
        }
    }
}

// ---- phase 1: tile reduction -------------------------------------------------
enum TileSrc { kTileF32 = 0, kTileBF16Fused = 1 };

struct TilePoolArgs {
    const void *feats;       // (B, N, C, H, W) f32 | bf16
    const void *weights;     // dist (B, N, D, H, W) f32 | logits bf16
    const uint4 *hdr;
    const uint32_t *rec;
    const uint4 *groups;
    const uint32_t *seg_row;
    float *rows;             // (B, max_seg, C)
    int64_t max_seg;
    TileGeom g;
    int C, wbudget;
};

// One union row of a group: acc[m][j] += (w[2m], w[2m+1]) * F[hl][lane + 32 j].
template <int CS, int FS>
__device__ __forceinline__ void group_row(float2 (&acc)[kTileGroup / 2][CS], const float *wq,
                                          const float *fs, int hl, int lane) {
    const float4 w0 = *reinterpret_cast<const float4 *>(wq);
    const float4 w1 = *reinterpret_cast<const float4 *>(wq + 4);
#pragma unroll
    for (int j = 0; j < CS; ++j) {
        const float f = fs[hl * FS + lane + 32 * j];
        ffma2(acc[0][j], make_float2(w0.x, w0.y), f);
        ffma2(acc[1][j], make_float2(w0.z, w0.w), f);
        ffma2(acc[2][j], make_float2(w1.x, w1.y), f);
        ffma2(acc[3][j], make_float2(w1.z, w1.w), f);
    }
}

template <int CS, int FS>
__device__ __forceinline__ void group_row2(float2 (&acc)[kTileGroup / 2][CS], const float *wq,
                                           const float *fs, int h0, int h1, int lane) {
    const float4 a0 = *reinterpret_cast<const float4 *>(wq);
    const float4 a1 = *reinterpret_cast<const float4 *>(wq + 4);
    const float4 b0 = *reinterpret_cast<const float4 *>(wq + kTileGroup);
    const float4 b1 = *reinterpret_cast<const float4 *>(wq + kTileGroup + 4);
    float fa[CS], fb[CS];
#pragma unroll
    for (int j = 0; j < CS; ++j) {
        fa[j] = fs[h0 * FS + lane + 32 * j];
        fb[j] = fs[h1 * FS + lane + 32 * j];
    }
#pragma unroll
    for (int j = 0; j < CS; ++j) {
        ffma2(acc[0][j], make_float2(a0.x, a0.y), fa[j]);
        ffma2(acc[1][j], make_float2(a0.z, a0.w), fa[j]);
        ffma2(acc[2][j], make_float2(a1.x, a1.y), fa[j]);
        ffma2(acc[3][j], make_float2(a1.z, a1.w), fa[j]);
    }
#pragma unroll
    for (int j = 0; j < CS; ++j) {
        ffma2(acc[0][j], make_float2(b0.x, b0.y), fb[j]);
        ffma2(acc[1][j], make_float2(b0.z, b0.w), fb[j]);
        ffma2(acc[2][j], make_float2(b1.x, b1.y), fb[j]);
        ffma2(acc[3][j], make_float2(b1.z, b1.w), fb[j]);
    }
}

// Every global load of a tile is independent of the others (the addresses
// follow from the tile index alone), so a CTA waits about one memory latency
// per stage: (1) the feature rows F[hl][c] and the depth weights w[hl][d] of
// the tile's pixels into shared memory -- for the fused variant the logits,
// soft-maxed in place -- (2) the records, which only index shared memory,
// aggregate the weights per (cell, row), (3) the group products.
template <int CS, int SRC, int CL>
__global__ void __launch_bounds__(kPoolThreads, 4)
tile_pool_kernel(TilePoolArgs a) {
    constexpr int CP = CS * 32;
    constexpr int FS = CP + 4;  // row stride: 16-byte aligned rows of channel quads
    constexpr int NW = kPoolThreads / 32;
    extern __shared__ __align__(16) float sm[];
    const TileGeom &g = a.g;
    const int64_t t = blockIdx.x;
    const int b = blockIdx.y;
    const TileId id = tile_id(t, g.W, g.n_hb, g.TH, g.H);
    const uint4 h = a.hdr[t];
    const int n_segs = int(h.y), n_groups = int(h.z);
    const int HW = g.H * g.W, C = a.C, D = g.D, PD = (D + 3) & ~3;
    float *ws = sm;                                           // weight window [wbudget]
    float *fs = ws + a.wbudget;                               // [TH][FS] feature rows
    float *pw = fs + g.TH * FS;                               // [TH][PD] depth weights
    const int64_t nb = int64_t(b) * g.N + id.n;
    const int64_t pix0 = int64_t(id.h0) * g.W + id.w;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the first RPT records of each thread are loaded now, beside the staging
    // (records [0, RPT * 256) cover the whole tile at the nuScenes shape)
    // the tile's group headers and segment-row indices (when they fit the
    // small caches) are copied to shared memory asynchronously now, so the
    // group products never wait on a global load
    __shared__ __align__(16) uint4 s_gt[kGtCache + 1];
    __shared__ uint32_t s_srow[kGtCache * kTileGroup];
    const bool gt_cached = n_groups <= kGtCache;
    if (gt_cached) {
        const uint4 *gsrc = a.groups + t * g.gcap;
        const uint32_t *ssrc = a.seg_row + t * g.tpc;
        for (int i = threadIdx.x; i <= n_groups; i += kPoolThreads)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(&s_gt[i]))),
                         "l"(gsrc + i));
        for (int i = threadIdx.x; i < n_segs; i += kPoolThreads)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(&s_srow[i]))),
                         "l"(ssrc + i));
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // distributed shared memory may be written only once every CTA of the
    // cluster is running: arrive now, wait just before the first remote store
    if (CL > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    // the first weight window's zeros (it is at most wbudget long; windows
    // are multiples of 8 floats: 16-byte stores), beside the staging
    for (uint32_t i = 4 * threadIdx.x; i < min(h.w, uint32_t(a.wbudget)); i += 4 * kPoolThreads)
        *reinterpret_cast<float4 *>(ws + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    constexpr int RPT = 16;
    const uint32_t *rt = a.rec + t * g.tpc;
    uint32_t pre[RPT];
    // (1) stage: F[hl][c] = features[n, c, h0 + hl, w]; w[hl][d] = dist[n, d, h0 + hl, w]
    // (stage_quads: cluster columns, distributed shared memory)
    {
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
        const int rank = CL > 1 ? int(cluster.block_rank()) : 0;
        const ColumnXfer x = column_xfer<CL>(rank, id.th, HW, g.W);
        float *rfs = CL > 1 ? cluster.map_shared_rank(fs, x.j) : fs;
        float *rpw = CL > 1 ? cluster.map_shared_rank(pw, x.j) : pw;
        const int64_t col = pix0 - rank + x.j;  // (h0, w_base + j)
        constexpr int ES = SRC == kTileF32 ? 4 : 2;
        // feature rows padded with zero channels up to CP (the products read
        // CS full channel slots)
        stage_quads<CL, ES>(x, a.feats, C, CP / 4, nb * C * HW + col, rfs, FS, true);
        stage_quads<CL, ES>(x, a.weights, D, (D + 3) >> 2, nb * D * HW + col, rpw, PD, false);
        // the first RPT records of each thread, in flight across the barrier
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const uint32_t k = threadIdx.x + kPoolThreads * u;
            pre[u] = k < h.x ? __ldg(rt + k) : 0u;
        }
        if (CL > 1)
            cluster.sync();
    }
    asm volatile("griddepcontrol.launch_dependents;");
    if (n_segs == 0) return;
    const uint4 *gt = gt_cached ? s_gt : a.groups + t * g.gcap;
    const uint32_t total_w = h.w;
    // fused: 1 / sum_d exp(l - max) of each pixel; the weights are left
    // unnormalised (exp2 of the scaled logits) and the aggregation scales
    // each (cell, row) sum by its row's factor
    __shared__ float s_inv[kTileMaxRows];
    if (SRC == kTileBF16Fused) {
        __syncthreads();
        // depth softmax of the tile's pixels (lift.py:17-31 semantics, fp32
        // from bf16 logits): 8 lanes per pixel, 4 pixels per warp at once
        // (pixel rows PD apart fall in distinct banks), lanes over depth bins
        constexpr float kLog2e = 1.4426950408889634f;
        const int sub = lane & 7;
        for (int hl0 = 4 * warp; hl0 < id.th; hl0 += 4 * NW) {
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
            if (on && sub == 0) s_inv[hl] = 1.f / sum;
        }
    }
    if (gt_cached) asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();  // every thread's copies visible (and the staging done)
    const uint32_t *srow = gt_cached ? s_srow : a.seg_row + t * g.tpc;
    float *rows = a.rows + int64_t(b) * a.max_seg * C;
    const int shift = g.hl_bits + g.d_bits;
    const uint32_t dmask = (1u << g.d_bits) - 1u, hmask = (1u << g.hl_bits) - 1u;
    const uint32_t wmask = (1u << (30 - shift)) - 1u;
    for (int q0 = 0; q0 < n_groups;) {
        // a window of groups whose weights fit the budget (one, for nearly
        // every tile: then no search)
        const uint4 G0 = q0 ? gt[q0] : make_uint4(0u, 0u, 0u, 0u);
        int q1 = n_groups;
        if (total_w - G0.z > uint32_t(a.wbudget)) {
            int lo = q0 + 1, hi = n_groups - 1;
            q1 = q0 + 1;  // one group always fits (8 x TH <= budget)
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
        const uint32_t wlen = w_end - G0.z;
        if (q0 > 0) {  // (the single / first window was zeroed before the staging)
            __syncthreads();  // previous window consumed
            for (uint32_t i = 4 * threadIdx.x; i < wlen; i += 4 * kPoolThreads)
                *reinterpret_cast<float4 *>(ws + i) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();  // staging done (first window) / window zeroed
        // (2) aggregate: each run of one (cell, row) summed in depth order
        // (records below RPT * 256 come from the prefetch)
        auto run = [&](uint32_t k, uint32_t r) {
            if (k < G0.w || k >= r_end || !(r >> 31)) return;
            const uint32_t widx = (r >> shift) & wmask, r0 = r;
            float sum = pw[((r >> g.d_bits) & hmask) * PD + (r & dmask)];
            for (uint32_t kk = k + 1; (r >> 30) & 1u; ++kk) {  // the run's later points
                r = __ldg(rt + kk);
                sum += pw[((r >> g.d_bits) & hmask) * PD + (r & dmask)];
            }
            if (SRC == kTileBF16Fused) sum *= s_inv[(r0 >> g.d_bits) & hmask];
            ws[widx - G0.z] = sum;
        };
#pragma unroll
        for (int u = 0; u < RPT; ++u) run(threadIdx.x + kPoolThreads * u, pre[u]);
        {
            constexpr int U = 4;
            // this thread's records k = threadIdx.x (mod 256) in [max(G0.w, RPT*256), r_end)
            uint32_t k_lo = max(G0.w, uint32_t(RPT * kPoolThreads));
            k_lo += (threadIdx.x - k_lo % kPoolThreads + kPoolThreads) % kPoolThreads;
            for (uint32_t k0 = k_lo; k0 < r_end; k0 += kPoolThreads * U) {
                uint32_t rr[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t k = k0 + kPoolThreads * u;
                    rr[u] = k < r_end ? __ldg(rt + k) : 0u;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) run(k0 + kPoolThreads * u, rr[u]);
            }
        }
        __syncthreads();
        // (3) one warp per group of 8 cells
        for (int q = q0 + warp; q < q1; q += NW) {
            const uint4 G = gt[q];
            // the group's segment-row indices, loaded before its products
            const int nk = min(kTileGroup, n_segs - q * kTileGroup);
            const uint32_t my_row = lane < nk ? srow[q * kTileGroup + lane] : 0u;
            const float *wq = ws + (G.z - G0.z);
            float2 acc[kTileGroup / 2][CS];
#pragma unroll
            for (int m = 0; m < kTileGroup / 2; ++m)
#pragma unroll
                for (int j = 0; j < CS; ++j) acc[m][j] = make_float2(0.f, 0.f);
            // rows two at a time: the second row's loads are in flight while
            // the first row's products issue
            for (int half = 0; half < 2; ++half) {
                uint32_t m = half ? G.y : G.x;
                const int base = half ? 31 : -1;
                if (m == 0xFFFFFFFFu) {  // all 32 rows (a level rig: most groups)
#pragma unroll 8
                    for (int h = base + 1; h < base + 33; h += 2) {
                        group_row2<CS, FS>(acc, wq, fs, h, h + 1, lane);
                        wq += 2 * kTileGroup;
                    }
                    continue;
                }
                while (m) {
                    const int h0 = base + __ffs(m);
                    m &= m - 1;
                    if (m) {
                        const int h1 = base + __ffs(m);
                        m &= m - 1;
                        group_row2<CS, FS>(acc, wq, fs, h0, h1, lane);
                        wq += 2 * kTileGroup;
                    } else {
                        group_row<CS, FS>(acc, wq, fs, h0, lane);
                        wq += kTileGroup;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kTileGroup; ++k) {
                const uint32_t row = __shfl_sync(0xFFFFFFFFu, my_row, k);
                if (k < nk) {
                    float *dst = rows + int64_t(row) * C;
#pragma unroll
                    for (int j = 0; j < CS; ++j) {
                        const int c = lane + 32 * j;
                        if (c < C) dst[c] = (k & 1) ? acc[k >> 1][j].y : acc[k >> 1][j].x;
                    }
                }
            }
        }
        q0 = q1;
    }
    __syncthreads();
}

// ---- phase 2: per-cell combine + transpose into the channel-major map -------
// A CTA owns 32 consecutive cells.  Warp w combines cells w, w+8, w+16, w+24
// with lanes over channels (a cell's segment rows are contiguous; one
// coalesced load per 32 channels of a row), into a shared [cell][channel]
// tile; then warp w writes channels w, w+8, ... of the 32 cells as full
// 128-byte lines.  Everything is 32-bit index math and fully unrolled over
// the channel slots: the kernel is bound by the map's stores.
template <int CS>
__global__ void __launch_bounds__(kPoolThreads)
tile_finalize_kernel(const float *__restrict__ rows, int64_t max_seg,
                     const uint32_t *__restrict__ cell_seg_first,
                     const uint32_t *__restrict__ cell_npts, int n_cells, int C, int mean,
                     float *__restrict__ out) {
    constexpr int CP = CS * 32;
    constexpr int NW = kPoolThreads / 32;
    __shared__ float tile[kFinCells][CP + 1];
    const int c0 = blockIdx.x * kFinCells, b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nc = min(kFinCells, n_cells - c0);
    const uint32_t f = __ldg(cell_seg_first + c0 + min(lane, nc));
    const uint32_t f_end = __ldg(cell_seg_first + c0 + nc);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // phase 1's rows (PDL)
    const float *rb = rows + int64_t(b) * max_seg * C;
#pragma unroll
    for (int u = 0; u < kFinCells / NW; ++u) {
        const int cl = warp + NW * u;
        const uint32_t s0 = __shfl_sync(0xFFFFFFFFu, f, cl);
        uint32_t s1 = cl < 31 ? __shfl_sync(0xFFFFFFFFu, f, cl + 1) : f_end;
        if (cl >= nc) s1 = s0;
        float acc[CS];
#pragma unroll
        for (int j = 0; j < CS; ++j) acc[j] = 0.f;
        if (s1 > s0) {
            const float *r = rb + int64_t(s0) * C + lane;
            const bool two = s1 > s0 + 1;  // ~22% of cells: load both rows at once
#pragma unroll
            for (int j = 0; j < CS; ++j)
                if (lane + 32 * j < C) {
                    acc[j] = __ldg(r + 32 * j);
                    if (two) acc[j] += __ldg(r + C + 32 * j);
                }
            r += C;
            for (uint32_t s = s0 + 2; s < s1; ++s) {
                r += C;
#pragma unroll
                for (int j = 0; j < CS; ++j)
                    if (lane + 32 * j < C) acc[j] += __ldg(r + 32 * j);
            }
            if (mean) {
                const float inv = 1.f / float(__ldg(cell_npts + c0 + cl));
#pragma unroll
                for (int j = 0; j < CS; ++j) acc[j] *= inv;
            }
        }
#pragma unroll
        for (int j = 0; j < CS; ++j) tile[cl][lane + 32 * j] = acc[j];
    }
    __syncthreads();
    if (lane < nc) {
        float *ob = out + int64_t(b) * C * n_cells + c0 + lane;
#pragma unroll
        for (int k = 0; k < CP / NW; ++k) {
            const int ch = warp + NW * k;
            if (ch < C) ob[int64_t(ch) * n_cells] = tile[lane][ch];
        }
    }
}

__global__ void tile_plan_count_kernel(const uint32_t *__restrict__ total, int64_t n_cells,
                                       uint32_t *__restrict__ csf, int64_t *__restrict__ nseg,
                                       const int *__restrict__ err) {
    csf[n_cells] = *total;
    nseg[0] = *err ? -1 : int64_t(*total);
}

template <int CS, int SRC, int CL>
static int launch_phase1(const TilePoolArgs &a, int B, size_t smem, cudaStream_t s) {
    static int max_dyn = -1;
    if (max_dyn < 0) {  // opt in to the full shared memory, less the static part
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, tile_pool_kernel<CS, SRC, CL>);
        max_dyn = 227 * 1024 - int(fa.sharedSizeBytes);
        cudaFuncSetAttribute(tile_pool_kernel<CS, SRC, CL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
    }
    BVP_REQUIRE(smem <= size_t(max_dyn), BVP_ERR_UNSUPPORTED,
                "tile needs %zu bytes of shared memory (max %d)", smem, max_dyn);
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
    const cudaError_t e = cudaLaunchKernelEx(&cfg, tile_pool_kernel<CS, SRC, CL>, a);
    BVP_REQUIRE(e == cudaSuccess, BVP_ERR_CUDA, "tile_pool launch: %s", cudaGetErrorString(e));
    return BVP_OK;
}

template <int CS, int SRC>
static int run_tile_pool(const void *feats, const void *weights, const bvp_tile_plan *p,
                         const TileGeom &g, int B, int C, int mean, int phases, float *rows,
                         float *out, cudaStream_t s) {
    const PlanLayout L = plan_layout(g, p->n_cells);
    TilePoolArgs a{};
    a.feats = feats;
    a.weights = weights;
    a.hdr = at<const uint4>(p, L.hdr);
    a.rec = at<const uint32_t>(p, L.rec);
    a.groups = at<const uint4>(p, L.groups);
    a.seg_row = at<const uint32_t>(p, L.seg_row);
    a.rows = rows;
    a.max_seg = p->max_seg;
    a.g = g;
    a.C = C;
    a.wbudget = std::max(2048, 128 * g.TH);
    const int CP = CS * 32;
    const size_t smem =
        sizeof(float) * (size_t(g.TH) * (CP + 4) + size_t(g.TH) * ((g.D + 3) & ~3) + a.wbudget);
    // clusters of CL adjacent columns (CL | W keeps a cluster inside one row
    // of tiles)
    int CL = (g.W % 8 == 0) ? 8 : (g.W % 4 == 0) ? 4 : (g.W % 2 == 0) ? 2 : 1;
    if (phases & 1) {
        int rc = BVP_OK;
        switch (CL) {
            case 8: rc = launch_phase1<CS, SRC, 8>(a, B, smem, s); break;
            case 4: rc = launch_phase1<CS, SRC, 4>(a, B, smem, s); break;
            case 2: rc = launch_phase1<CS, SRC, 2>(a, B, smem, s); break;
            default: rc = launch_phase1<CS, SRC, 1>(a, B, smem, s); break;
        }
        if (rc != BVP_OK) return rc;
    }
    if (phases & 2) {
        // programmatic dependent launch: the combine's CTAs take the slots
        // phase-1 CTAs free, read their cell tables, and wait in
        // griddepcontrol.wait until phase 1's rows are complete
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(ceil_div(p->n_cells, kFinCells)), unsigned(B));
        cfg.blockDim = dim3(kPoolThreads);
        cfg.stream = s;
        cudaLaunchAttribute at1[1];
        at1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at1[0].val.programmaticStreamSerializationAllowed = (phases & 1) ? 1 : 0;
        cfg.attrs = at1;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(
            &cfg, tile_finalize_kernel<CS>, static_cast<const float *>(rows), p->max_seg,
            at<const uint32_t>(p, L.csf), at<const uint32_t>(p, L.npts), int(p->n_cells), C, mean,
            out);
        BVP_REQUIRE(e == cudaSuccess, BVP_ERR_CUDA, "tile_finalize launch: %s",
                    cudaGetErrorString(e));
    }
    return check_launch("tile_pool");
}

template <int SRC>
static int tile_pool_dispatch(const void *feats, const void *weights, const bvp_tile_plan *p,
                              int B, int C, int mode, float *rows, size_t rows_bytes, float *out,
                              cudaStream_t s) {
    TileGeom g;
    const int rc = plan_dims_from(p, g);
    if (rc != BVP_OK) return rc;
    BVP_REQUIRE(B >= 1 && C >= 0, BVP_ERR_INVALID, "bad dims B=%d C=%d", B, C);
    int phases = 3;
    if (mode & (BVP_TILE_PHASE1 | BVP_TILE_PHASE2))
        phases = ((mode & BVP_TILE_PHASE1) ? 1 : 0) | ((mode & BVP_TILE_PHASE2) ? 2 : 0);
    mode &= ~(BVP_TILE_PHASE1 | BVP_TILE_PHASE2);
    BVP_REQUIRE(mode == BVP_SUM || mode == BVP_MEAN, BVP_ERR_UNSUPPORTED,
                "the tile path reduces SUM and MEAN only (mode %d)", mode);
    BVP_REQUIRE(C <= 128, BVP_ERR_UNSUPPORTED, "the tile path takes C <= 128 (C=%d)", C);
    if (C == 0) return BVP_OK;
    BVP_REQUIRE(feats && weights && out && rows, BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(rows_bytes >= size_t(B) * p->max_seg * C * sizeof(float), BVP_ERR_INVALID,
                "segment-row scratch too small: need %zu bytes, got %zu",
                size_t(B) * p->max_seg * C * sizeof(float), rows_bytes);
    const int mean = mode == BVP_MEAN;
    switch ((C + 31) / 32) {
        case 1: return run_tile_pool<1, SRC>(feats, weights, p, g, B, C, mean, phases, rows, out, s);
        case 2: return run_tile_pool<2, SRC>(feats, weights, p, g, B, C, mean, phases, rows, out, s);
        case 3: return run_tile_pool<3, SRC>(feats, weights, p, g, B, C, mean, phases, rows, out, s);
        default: return run_tile_pool<4, SRC>(feats, weights, p, g, B, C, mean, phases, rows, out, s);
    }
}

}  // namespace bvp

using namespace bvp;

extern "C" {

int bvp_tile_plan_supported(int N, int H, int W, int D, int64_t n_cells) {
    return plan_supported(N, H, W, D, n_cells) ? 1 : 0;
}

size_t bvp_tile_plan_bytes(int N, int H, int W, int D, int64_t n_cells) {
    if (!plan_supported(N, H, W, D, n_cells)) return 0;
    return plan_layout(tile_geom(N, H, W, D), n_cells).bytes;
}

size_t bvp_tile_plan_workspace_bytes(int N, int H, int W, int D, int64_t n_cells) {
    if (!plan_supported(N, H, W, D, n_cells)) return 0;
    return plan_ws(tile_geom(N, H, W, D), n_cells).bytes;
}

static int build_tile_plan(const uint32_t *cell_of_point, const uint32_t *ranks,
                           const int64_t *counts, bvp_tile_plan *plan, void *workspace,
                           size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(cell_of_point, BVP_ERR_INVALID, "null cell_of_point");
    BVP_REQUIRE((ranks == nullptr) == (counts == nullptr), BVP_ERR_INVALID,
                "ranks and counts go together");
    TileGeom g;
    int rc = plan_dims_from(plan, g);
    if (rc != BVP_OK) return rc;
    const int64_t n_cells = plan->n_cells;
    const PlanLayout L = plan_layout(g, n_cells);
    const PlanWs WL = plan_ws(g, n_cells);
    BVP_REQUIRE(plan->bytes >= L.bytes, BVP_ERR_INVALID, "tile plan buffer too small");
    BVP_REQUIRE(workspace && workspace_bytes >= WL.bytes, BVP_ERR_INVALID,
                "tile plan workspace too small: need %zu bytes, got %zu", WL.bytes,
                workspace_bytes);
    cudaStream_t s = as_stream(stream);
    char *w = static_cast<char *>(workspace);
    auto *fill = reinterpret_cast<uint32_t *>(w + WL.fill);
    auto *owner = reinterpret_cast<unsigned long long *>(w + WL.owner);
    auto *part = reinterpret_cast<uint32_t *>(w + WL.part);
    auto *total = reinterpret_cast<uint32_t *>(w + WL.total);
    auto *err = reinterpret_cast<int *>(w + WL.err);
    auto *csf = at<uint32_t>(plan, L.csf);
    auto *npts = at<uint32_t>(plan, L.npts);
    cudaMemsetAsync(err, 0, 8, s);
    cudaMemsetAsync(csf, 0, 4 * size_t(n_cells + 1), s);
    cudaMemsetAsync(npts, 0, 4 * size_t(n_cells), s);
    cudaMemsetAsync(fill, 0, 4 * size_t(n_cells + 1), s);
    int cap = 1;
    while (cap < g.tpc) cap <<= 1;
    const size_t smem = 8 * size_t(cap);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tile_plan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             8 * kTileMaxPoints);
        cudaFuncSetAttribute(tile_plan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             8 * kTileMaxPoints);
        attr = true;
    }
    TileSorted ts{};
    // (the per-tile histogram lives in shared memory: up to 12288 tiles)
    if (ranks && g.T * 4 > 48 * 1024) ranks = nullptr;
    if (ranks) {  // the tiles' points in order from the association: a stable partition
        const int64_t P = int64_t(g.N) * g.H * g.W * g.D;
        auto *tkeys = reinterpret_cast<uint32_t *>(w + WL.tkeys);
        auto *tpts = reinterpret_cast<uint32_t *>(w + WL.tpts);
        auto *tstart = reinterpret_cast<uint32_t *>(w + WL.tstart);
        cudaMemsetAsync(tstart, 0, 4 * size_t(g.T + 1), s);
        const unsigned kb = unsigned(std::min<int64_t>(ceil_div(P, 256), 148 * 4));
        tile_key_kernel<<<kb, 256, 4 * size_t(g.T), s>>>(ranks, counts, g, P, tkeys, tstart);
        device_excl_scan<uint32_t>(tstart, tstart, g.T + 1, reinterpret_cast<uint32_t *>(w + WL.tpart),
                                   reinterpret_cast<uint32_t *>(w + WL.ttotal), s);
        rc = stable_partition(tkeys, ranks, counts, P, bits_for(g.T - 1), tpts, w + WL.tsort,
                              WL.tsort_bytes, s);
        if (rc != BVP_OK) return rc;
        ts = TileSorted{tpts, tstart};
        tile_plan_kernel<true><<<unsigned(g.T), kPlanThreads, smem, s>>>(
            cell_of_point, g, at<uint4>(plan, L.hdr), at<uint32_t>(plan, L.rec),
            at<uint32_t>(plan, L.seg_cell), at<uint32_t>(plan, L.seg_start),
            at<uint4>(plan, L.groups), err, ts);
    } else {
        tile_plan_kernel<false><<<unsigned(g.T), kPlanThreads, smem, s>>>(
            cell_of_point, g, at<uint4>(plan, L.hdr), at<uint32_t>(plan, L.rec),
            at<uint32_t>(plan, L.seg_cell), at<uint32_t>(plan, L.seg_start),
            at<uint4>(plan, L.groups), err, ts);
    }
    tile_seg_count_kernel<<<unsigned(g.T), 256, 0, s>>>(
        at<const uint4>(plan, L.hdr), g, at<const uint32_t>(plan, L.seg_cell),
        at<const uint32_t>(plan, L.seg_start), csf, npts);
    device_excl_scan<uint32_t>(csf, csf, n_cells, part, total, s);
    tile_plan_count_kernel<<<1, 1, 0, s>>>(total, n_cells, csf, at<int64_t>(plan, L.nseg), err);
    tile_seg_assign_kernel<<<unsigned(g.T), 256, 0, s>>>(at<const uint4>(plan, L.hdr), g,
                                                          at<const uint32_t>(plan, L.seg_cell),
                                                          csf, fill, owner);
    const unsigned cb = unsigned(std::min<int64_t>(ceil_div(n_cells, 256), 148 * 16));
    tile_seg_fix_kernel<<<cb, 256, 0, s>>>(csf, n_cells, g, owner, at<uint32_t>(plan, L.seg_row));
    return check_launch("build_tile_plan");
}

int bvp_build_tile_plan(const uint32_t *cell_of_point, bvp_tile_plan *plan, void *workspace,
                        size_t workspace_bytes, void *stream) {
    return build_tile_plan(cell_of_point, nullptr, nullptr, plan, workspace, workspace_bytes,
                           stream);
}

int bvp_build_tile_plan_ranks(const uint32_t *cell_of_point, const uint32_t *ranks,
                              const int64_t *counts, bvp_tile_plan *plan, void *workspace,
                              size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(ranks && counts, BVP_ERR_INVALID, "null ranks / counts");
    return build_tile_plan(cell_of_point, ranks, counts, plan, workspace, workspace_bytes,
                           stream);
}

int bvp_tile_plan_init(bvp_tile_plan *plan, int N, int H, int W, int D, int64_t n_cells,
                       void *base, size_t bytes, int64_t max_seg) {
    BVP_REQUIRE(plan, BVP_ERR_INVALID, "null plan");
    BVP_REQUIRE(plan_supported(N, H, W, D, n_cells), BVP_ERR_UNSUPPORTED,
                "frustum %dx%dx%dx%d / %lld cells not supported by the tile plan", N, H, W, D,
                (long long)n_cells);
    const TileGeom g = tile_geom(N, H, W, D);
    const PlanLayout L = plan_layout(g, n_cells);
    BVP_REQUIRE(base && bytes >= L.bytes, BVP_ERR_INVALID, "tile plan buffer too small");
    plan->N = N; plan->H = H; plan->W = W; plan->D = D;
    plan->n_cells = n_cells;
    plan->base = base;
    plan->bytes = bytes;
    plan->max_seg = max_seg;
    plan->tile_rows = g.TH;
    plan->n_tiles = g.T;
    plan->n_seg = reinterpret_cast<const int64_t *>(static_cast<char *>(base) + L.nseg);
    plan->cell_seg_first = reinterpret_cast<const uint32_t *>(static_cast<char *>(base) + L.csf);
    plan->cell_points = reinterpret_cast<const uint32_t *>(static_cast<char *>(base) + L.npts);
    return BVP_OK;
}

int bvp_tile_pool_f32(const float *features, const float *dist, const bvp_tile_plan *plan, int B,
                      int C, int mode, float *rows, size_t rows_bytes, float *out, void *stream) {
    return tile_pool_dispatch<kTileF32>(features, dist, plan, B, C, mode, rows, rows_bytes, out,
                                        as_stream(stream));
}


int bvp_tile_pool_fused_bf16(const uint16_t *logits, const uint16_t *context,
                             const bvp_tile_plan *plan, int B, int C, int mode, float *rows,
                             size_t rows_bytes, float *out, void *stream) {
    return tile_pool_dispatch<kTileBF16Fused>(context, logits, plan, B, C, mode, rows, rows_bytes,
                                              out, as_stream(stream));
}

}  // extern "C"

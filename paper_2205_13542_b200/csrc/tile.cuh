// tile.cuh -- shared by the tiled reduction (tile.cu) and its adjoint
// (tile_backward.cu): tile geometry, plan layout, cluster column staging.
#pragma once

#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"
#include "partition.cuh"
#include "scan.cuh"

namespace bvp {

constexpr int kTileGroup = 8;         // segments (cells) per group
constexpr int kTileMaxRows = 64;      // rows per tile (one u64 mask per group)
constexpr int kTileRows = 32;         // rows per tile chosen (tile_rows_for)
constexpr int kTileMaxPoints = 8192;  // points per tile (smem sort capacity)
constexpr int kPlanThreads = 512;
constexpr int kPoolThreads = 256;
constexpr int kFinCells = 32;         // cells per finalize CTA
constexpr int kGtCache = 32;          // group headers cached in shared memory

struct TileGeom {
    int N, H, W, D, TH, n_hb;
    int64_t T, tpc, gcap;
    int hl_bits, d_bits;
};

inline int bits_for(int64_t v) {  // bits to hold values in [0, v]
    int b = 0;
    while (b < 62 && (int64_t(1) << b) <= v) ++b;
    return b;
}

// Rows per tile: at most kTileRows (measured at config H, 64 rows: 32-row
// tiles take the step from 203 to 178 us -- four 45 KB CTAs per SM instead
// of two 88 KB ones outweigh twice the segment rows; 16 or 24 rows are
// slower), balanced over the fewest row blocks, and at most kTileMaxPoints
// points per tile.
inline int tile_rows_for(int H, int D) {
    const int cap = std::min(kTileRows, std::max(1, kTileMaxPoints / std::max(D, 1)));
    const int n_hb = (H + cap - 1) / cap;
    return (H + n_hb - 1) / n_hb;
}

inline TileGeom tile_geom(int N, int H, int W, int D) {
    TileGeom g{};
    g.N = N; g.H = H; g.W = W; g.D = D;
    g.TH = tile_rows_for(H, D);
    g.n_hb = int((H + g.TH - 1) / g.TH);
    g.T = int64_t(N) * g.n_hb * W;
    g.tpc = int64_t(g.TH) * D;
    g.gcap = (g.tpc + kTileGroup - 1) / kTileGroup + 1;  // + sentinel
    g.hl_bits = bits_for(g.TH - 1);
    g.d_bits = bits_for(D - 1);
    return g;
}

// tile index t = (n * n_hb + hb) * W + w: neighbouring columns are
// neighbouring tiles, so concurrently running CTAs share the 32-byte sectors
// of the strided (N, C, H, W) / (N, D, H, W) inputs through L2.
struct TileId {
    int n, hb, w, h0, th;
};
__device__ __forceinline__ TileId tile_id(int64_t t64, int W, int n_hb, int TH, int H) {
    TileId r;
    const int t = int(t64);  // T < 2^31 (plan_supported)
    r.w = t % W;
    const int rest = t / W;
    r.hb = rest % n_hb;
    r.n = rest / n_hb;
    r.h0 = r.hb * TH;
    r.th = min(TH, H - r.h0);
    return r;
}

// ---- block helpers ---------------------------------------------------------
// Exclusive scan of one value per thread across the block (blockDim.x <= 1024).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *s_warp,
                                                    uint32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t y = lane < nw ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t z = __shfl_up_sync(0xFFFFFFFFu, y, o);
            if (lane >= o) y += z;
        }
        if (lane < nw) s_warp[lane] = y;  // inclusive warp totals
    }
    __syncthreads();
    const uint32_t pre = warp ? s_warp[warp - 1] : 0u;
    if (total) *total = s_warp[nw - 1];
    __syncthreads();
    return pre + x - v;
}


// acc.x += w.x * f, acc.y += w.y * f in one FFMA2 (Blackwell packed fp32;
// the scalar f is a broadcast operand, no move).
__device__ __forceinline__ void ffma2(float2 &acc, float2 w, float f) {
    unsigned long long a = *reinterpret_cast<unsigned long long *>(&acc);
    const unsigned long long wv = *reinterpret_cast<const unsigned long long *>(&w);
    unsigned long long fv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(fv) : "f"(f));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(wv), "l"(fv));
    acc = *reinterpret_cast<float2 *>(&a);
}

// ---- cluster column staging ---------------------------------------------------
// The CL tiles of a cluster are CL adjacent columns of one camera.  CTA
// `rank` moves channel quads (and depth-bin quads) rank, rank + CL, ... for
// all CL columns -- a warp's access covers CL neighbouring columns x 32/CL
// rows, 32/CL lines instead of 32 -- each quad one 16-byte word in the
// shared memory of the CTA owning its column (distributed shared memory).
struct ColumnXfer {
    int rank, j, r0;  // this CTA's rank; the lane's column (peer) and first row
    int n_rb, th;     // row blocks of 32/CL rows; rows of the tile
    int HW, W;
};

template <int CL>
__device__ __forceinline__ ColumnXfer column_xfer(int rank, int th, int HW, int W) {
    const int lane = threadIdx.x & 31;
    constexpr int RS = 32 / CL;
    return ColumnXfer{rank, lane % CL, lane / CL, (th + RS - 1) / RS, th, HW, W};
}

// item it = (quad qi, row block m); the U items of a round are NW apart, so
// one division per round and carries after it
template <int U>
__device__ __forceinline__ void xfer_items(int i0, int n_rb, int (&qs)[U], int (&ms)[U]) {
    constexpr int NW = kPoolThreads / 32;
    int qi = i0 / n_rb, m = i0 - qi * n_rb;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        qs[u] = qi;
        ms[u] = m;
        m += NW;
        while (m >= n_rb) {
            m -= n_rb;
            ++qi;
        }
    }
}

// Global -> (remote) shared: rows [0, th) x quads of src (planes HW apart,
// column base `base` of the cluster's first column + j) into dst[hl][c]
// (stride floats).  n_quads >= ceil(n_ch / 4): quads past n_ch are stored as
// zeros.  ES: element bytes (4 fp32, 2 bf16 widened).  wait_first: the
// cluster barrier's wait (every CTA running, so its shared memory may be
// written) sits between the first round's loads and its stores.
template <int CL, int ES>
__device__ __forceinline__ void stage_quads(const ColumnXfer &x, const void *src, int n_ch,
                                            int n_quads, int64_t base, float *dst, int stride,
                                            bool wait_first) {
    constexpr int NW = kPoolThreads / 32, RS = 32 / CL, U = 4;
    const int warp = threadIdx.x >> 5;
    // byte addresses: the tile's column once, then one 32-bit offset per item
    // and one add per channel of the quad
    const char *sb = static_cast<const char *>(src) + base * ES;
    const uint32_t plane = uint32_t(x.HW) * ES, rowb = uint32_t(x.W) * ES;
    const int n_q = (n_quads - x.rank + CL - 1) / CL;  // this CTA's quads
    const int items = n_q * x.n_rb;
    for (int i0 = warp; i0 < items || (wait_first && i0 == warp); i0 += NW * U) {
        int qs[U], ms[U];
        xfer_items<U>(i0, x.n_rb, qs, ms);
        // all U x 4 loads issue before any value is used (raw bits; bf16
        // widened at the store)
        uint32_t v[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int it = i0 + NW * u;
            const int c0 = 4 * (x.rank + CL * qs[u]), hl = x.r0 + RS * ms[u];
            const bool ok = it < items && hl < x.th;
            const char *pi = sb + (uint64_t(uint32_t(c0)) * plane + uint32_t(hl) * rowb);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const bool on = ok && c0 + e < n_ch;
                if (ES == 4)
                    v[u][e] = ldg_l2pf_b32(pi + uint64_t(e) * plane, on);
                else
                    v[u][e] = ldg_l2pf_u16(pi + uint64_t(e) * plane, on) << 16;
            }
        }
        if (CL > 1 && wait_first && i0 == warp)
            asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int it = i0 + NW * u;
            const int c0 = 4 * (x.rank + CL * qs[u]), hl = x.r0 + RS * ms[u];
            if (it < items && hl < x.th)
                *reinterpret_cast<float4 *>(dst + hl * stride + c0) =
                    make_float4(__uint_as_float(v[u][0]), __uint_as_float(v[u][1]),
                                __uint_as_float(v[u][2]), __uint_as_float(v[u][3]));
        }
    }
}

// (Remote) shared -> global, the reverse of stage_quads: src[hl][c] of the
// CTA owning column j into dst planes (fp32, or bf16 rounded to nearest),
// channels < n_ch.
__device__ __forceinline__ void store_as(float *p, float v) { *p = v; }
__device__ __forceinline__ void store_as(__nv_bfloat16 *p, float v) { *p = __float2bfloat16(v); }
template <int CL, typename OT = float>
__device__ __forceinline__ void unstage_quads(const ColumnXfer &x, OT *dst, int n_ch,
                                              int64_t base, const float *src, int stride) {
    constexpr int NW = kPoolThreads / 32, RS = 32 / CL, U = 4;
    const int warp = threadIdx.x >> 5;
    OT *db = dst + base;
    const int n_q = (((n_ch + 3) >> 2) - x.rank + CL - 1) / CL;
    const int items = n_q * x.n_rb;
    for (int i0 = warp; i0 < items; i0 += NW * U) {
        int qs[U], ms[U];
        xfer_items<U>(i0, x.n_rb, qs, ms);
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int it = i0 + NW * u;
            const int c0 = 4 * (x.rank + CL * qs[u]), hl = x.r0 + RS * ms[u];
            v[u] = it < items && hl < x.th
                       ? *reinterpret_cast<const float4 *>(src + hl * stride + c0)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int it = i0 + NW * u;
            const int c0 = 4 * (x.rank + CL * qs[u]), hl = x.r0 + RS * ms[u];
            if (it < items && hl < x.th) {
                OT *po = db + int64_t(c0) * x.HW + int64_t(hl) * x.W;
                const float e4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (c0 + e < n_ch) store_as(po + int64_t(e) * x.HW, e4[e]);
            }
        }
    }
}

// ---- plan layout -------------------------------------------------------------
static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

struct PlanLayout {
    size_t hdr, rec, seg_cell, seg_start, seg_row, groups, csf, npts, nseg, bytes;
};
static PlanLayout plan_layout(const TileGeom &g, int64_t n_cells) {
    PlanLayout L{};
    size_t o = 0;
    const size_t pts = size_t(g.T) * g.tpc;
    L.hdr = o; o = a256(o + 16 * size_t(g.T));
    L.rec = o; o = a256(o + 4 * pts);
    L.seg_cell = o; o = a256(o + 4 * pts);
    L.seg_start = o; o = a256(o + 4 * pts);
    L.seg_row = o; o = a256(o + 4 * pts);
    L.groups = o; o = a256(o + 16 * size_t(g.T) * g.gcap);
    L.csf = o; o = a256(o + 4 * size_t(n_cells + 1));
    L.npts = o; o = a256(o + 4 * size_t(n_cells));
    L.nseg = o; o = a256(o + 8);
    L.bytes = o;
    return L;
}

struct PlanWs {
    size_t fill, owner, part, total, err;
    // the by-tile partition of the association's ranks (bvp_build_tile_plan_ranks)
    size_t tkeys, tpts, tstart, tpart, ttotal, tsort, tsort_bytes, bytes;
};
static PlanWs plan_ws(const TileGeom &g, int64_t n_cells) {
    PlanWs L{};
    const int64_t P = int64_t(g.N) * g.H * g.W * g.D;
    size_t o = 0;
    L.fill = o; o = a256(o + 4 * size_t(n_cells + 1));
    L.owner = o; o = a256(o + 8 * size_t(g.T) * g.tpc);
    L.part = o; o = a256(o + 4 * size_t(scan_partials_len<uint32_t>(n_cells + 1)));
    L.total = o; o = a256(o + 8);
    L.err = o; o = a256(o + 8);
    L.tkeys = o; o = a256(o + 4 * size_t(P));
    L.tpts = o; o = a256(o + 4 * size_t(P));
    L.tstart = o; o = a256(o + 4 * size_t(g.T + 1));
    L.tpart = o; o = a256(o + 4 * size_t(scan_partials_len<uint32_t>(g.T + 1)));
    L.ttotal = o; o = a256(o + 8);
    L.tsort_bytes = stable_partition_ws_bytes(P, bits_for(g.T - 1));
    L.tsort = o; o = a256(o + L.tsort_bytes);
    L.bytes = o;
    return L;
}


static bool plan_supported(int N, int H, int W, int D, int64_t n_cells) {
    if (N < 1 || H < 1 || W < 1 || D < 1 || D > kTileMaxPoints) return false;
    if (n_cells < 1 || n_cells >= (int64_t(1) << 31) - 32) return false;
    const TileGeom g = tile_geom(N, H, W, D);
    return g.T < (int64_t(1) << 31) && g.tpc <= kTileMaxPoints &&
           g.hl_bits + g.d_bits <= 16;
}

static int plan_dims_from(const bvp_tile_plan *p, TileGeom &g) {
    BVP_REQUIRE(p && p->base, BVP_ERR_INVALID, "null tile plan");
    BVP_REQUIRE(plan_supported(p->N, p->H, p->W, p->D, p->n_cells), BVP_ERR_UNSUPPORTED,
                "frustum %dx%dx%dx%d not supported by the tile plan", p->N, p->H, p->W, p->D);
    g = tile_geom(p->N, p->H, p->W, p->D);
    return BVP_OK;
}

template <typename T>
static T *at(const bvp_tile_plan *p, size_t off) {
    return reinterpret_cast<T *>(static_cast<char *>(p->base) + off);
}

}  // namespace bvp

// work.cu -- the chunk schedule of the fast interval kernel (pool_ivl.cuh),
// part of the cached association (built once per rig, like the ranks).
//
// Every interval of the reference's interval table (bevgrid.py:142-158) is
// cut into chunks of <= chunk consecutive sorted points.  The kernel gives
// each chunk to one lane group, which sums it sequentially; chunks are
// listed longest first so the 8 groups of a warp run for the same number of
// steps (measured 99.9% group utilisation at the nuScenes shape, vs 43% for
// one group per cell of an 8-cell row tile).  A chunk of an interval that
// was NOT cut writes its cell directly; chunks of a cut ("split") interval
// write fp32 partials that a second pass adds in chunk order.
//
// work[4 w..]:  first sorted point, end, destination, interval (split chunks:
//               split index).  destination: the cell id, or kSplitDest |
//               partial slot
// splits[4 s..]: interval, cell, first partial slot, chunk count
// counts:       n_work, n_splits, n_partials
//
// The order of chunks of equal length is whatever the atomics produce; it
// changes no output bit (every chunk is summed by one group in rank order and
// partials are combined in slot order).
//
// The point gather table (point_meta) turns every sorted point's id into its
// feature row and weight index once, so the interval kernels never divide.
#include <algorithm>

#include "scan.cuh"

namespace bvp {

constexpr uint32_t kSplitDest = 0x80000000u;

// per interval: (chunk count, partial count (chunks if split), split flag, 0)
// -- one uint4 so a single scan yields all three bases
__global__ void work_count_kernel(const uint32_t *__restrict__ starts,
                                  const int64_t *__restrict__ counts, int64_t n_int_max,
                                  uint32_t chunk, uint4 *__restrict__ cnt) {
    const int64_t n_int = counts[1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_int_max;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        if (i < n_int) c = (starts[i + 1] - starts[i] + chunk - 1) / chunk;
        cnt[i] = make_uint4(c, c > 1 ? c : 0u, c > 1 ? 1u : 0u, 0u);
    }
}

// per interval: emit its chunks (unsorted, chunk order) with a length
// histogram; splits table
__global__ void work_emit_kernel(const uint32_t *__restrict__ starts,
                                 const uint32_t *__restrict__ icells,
                                 const int64_t *__restrict__ counts, uint32_t chunk,
                                 const uint4 *__restrict__ base, uint4 *__restrict__ tmp,
                                 uint32_t *__restrict__ keys, uint4 *__restrict__ splits,
                                 int ny, int tile) {
    const int tiles_y = tile > 0 ? (ny + tile - 1) / tile : 1;
    const int64_t n_int = counts[1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_int;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t lo = starts[i], hi = starts[i + 1], cell = icells[i];
        const uint32_t nch = (hi - lo + chunk - 1) / chunk;
        const uint4 b = base[i];  // exclusive: chunk, partial, split bases
        const bool split = nch > 1;
        for (uint32_t k = 0; k < nch; ++k) {
            const uint32_t a = lo + k * chunk, e = min(hi, a + chunk);
            const uint32_t dest = split ? (kSplitDest | (b.y + k)) : cell;
            // .w: the interval, or for a chunk of a split interval its split index
            tmp[b.x + k] = make_uint4(a, e, dest, split ? b.z : static_cast<uint32_t>(i));
            // bucket 0 = longest; tile > 0: 2D cell tiles first (L1 reuse of
            // the feature rows shared by neighbouring cells), length within
            uint32_t key = chunk - (e - a);
            if (tile > 0) {
                const uint32_t ix = cell / uint32_t(ny), iy = cell - ix * uint32_t(ny);
                key += (chunk + 1) * ((ix / tile) * tiles_y + iy / tile);
            }
            if (keys) keys[b.x + k] = key;
        }
        if (split) splits[b.z] = make_uint4(static_cast<uint32_t>(i), cell, b.y, nch);
    }
}

// keys of the unused tail: out of range (dropped by the sort)
__global__ void work_keys_tail_kernel(const uint32_t *__restrict__ n_work_p, int64_t cap,
                                      uint32_t *__restrict__ keys) {
    const int64_t n = *n_work_p;
    for (int64_t w = n + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < cap;
         w += (int64_t)gridDim.x * blockDim.x)
        keys[w] = BVP_OUT_OF_RANGE;
}

__global__ void work_gather_kernel(const uint4 *__restrict__ tmp, const uint32_t *__restrict__ order,
                                   const uint32_t *__restrict__ n_work_p, uint4 *__restrict__ work) {
    const int64_t n = *n_work_p;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n;
         w += (int64_t)gridDim.x * blockDim.x)
        work[w] = tmp[order[w]];
}

__global__ void work_counts_kernel(const uint4 *__restrict__ tot, int64_t *__restrict__ out) {
    const uint4 t = *tot;
    out[0] = t.x;  // chunks
    out[1] = t.z;  // split intervals
    out[2] = t.y;  // partials
}

// Per sorted point: (feature row = pixel, weight index into (N,D,H,W)).
__global__ void point_meta_kernel(const uint32_t *__restrict__ ranks,
                                  const int64_t *__restrict__ counts, int64_t P, int D, int HW,
                                  uint2 *__restrict__ meta) {
    const int64_t n_in = counts[0];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_in && j < P;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = ranks[j];
        const uint32_t pix = p / D, d = p - pix * D;
        const uint32_t n = pix / HW, hw = pix - n * HW;
        meta[j] = make_uint2(pix, (n * D + d) * HW + hw);
    }
}

struct WorkLayout {
    size_t off_cnt, off_part, off_tot, off_tmp, off_keys, off_order,
        off_sstarts, off_scells, off_sfirst, off_scounts, off_sws, sort_ws, bytes;
};
static int64_t work_cap(int64_t n_int_max, int64_t n_points, int chunk) {
    return chunk > 0 ? n_int_max + n_points / chunk + 1 : 0;
}
static int64_t work_keys(int chunk, int nx, int ny, int tile) {
    if (tile < 0) return 1;  // unsorted: no sort workspace
    const int64_t nt = tile > 0 ? int64_t((nx + tile - 1) / tile) * ((ny + tile - 1) / tile) : 1;
    return nt * (chunk + 1);
}
static WorkLayout work_layout(int64_t n_int_max, int64_t n_points, int chunk, int64_t nkeys) {
    WorkLayout L{};
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t n = size_t(n_int_max);
    const int64_t cap = work_cap(n_int_max, n_points, chunk);
    size_t o = 0;
    L.off_cnt = o; o = al(o + n * 16);
    L.off_part = o; o = al(o + size_t(scan_partials_len<uint4>(n_int_max)) * 16);
    L.off_tot = o; o = al(o + 16);
    L.off_tmp = o; o = al(o + size_t(cap) * 16);
    L.off_keys = o; o = al(o + size_t(cap) * 4);
    L.off_order = o; o = al(o + size_t(cap) * 4);
    L.off_sstarts = o; o = al(o + size_t(nkeys + 1) * 4);
    L.off_scells = o; o = al(o + size_t(nkeys + 1) * 4);
    L.off_sfirst = o; o = al(o + size_t(nkeys + 1) * 4);
    L.off_scounts = o; o = al(o + 16);
    L.sort_ws = bvp_sort_workspace_bytes(cap, nkeys);
    L.off_sws = o; o = al(o + L.sort_ws);
    L.bytes = o;
    return L;
}

}  // namespace bvp

using namespace bvp;

extern "C" {

int bvp_point_meta(const uint32_t *ranks, const int64_t *counts, int N, int H, int W, int D,
                   uint32_t *point_meta, void *stream) {
    BVP_REQUIRE(ranks && counts && point_meta, BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(N >= 1 && H >= 1 && W >= 1 && D >= 1, BVP_ERR_INVALID, "bad dims");
    const int64_t P = int64_t(N) * H * W * D;
    const unsigned mb = static_cast<unsigned>(std::min<int64_t>(ceil_div(P, 256), int64_t(148) * 32));
    point_meta_kernel<<<mb, 256, 0, as_stream(stream)>>>(ranks, counts, P, D, H * W,
                                                         reinterpret_cast<uint2 *>(point_meta));
    return check_launch("point_meta");
}

int64_t bvp_work_capacity(int64_t n_int_max, int64_t n_points, int chunk) {
    return work_cap(n_int_max, n_points, chunk);
}

size_t bvp_work_workspace_bytes(int64_t n_int_max, int64_t n_points, int chunk, int nx, int ny,
                                int tile) {
    return work_layout(n_int_max, n_points, chunk, work_keys(chunk, nx, ny, tile)).bytes;
}

int bvp_make_work(const uint32_t *interval_starts, const uint32_t *interval_cells,
                  const int64_t *counts, int64_t n_int_max, int64_t n_points, int chunk,
                  int nx, int ny, int tile, uint32_t *work, uint32_t *splits,
                  int64_t *work_counts, void *workspace, size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(interval_starts && interval_cells && counts && work && splits && work_counts,
                BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(chunk >= 1 && chunk <= 4096 && n_int_max >= 1 && n_points >= 1, BVP_ERR_INVALID,
                "bad chunk %d or sizes", chunk);
    BVP_REQUIRE(nx >= 1 && ny >= 1 && tile >= -1, BVP_ERR_INVALID, "bad grid / tile");
    const int64_t nkeys = work_keys(chunk, nx, ny, tile);
    const WorkLayout L = work_layout(n_int_max, n_points, chunk, nkeys);
    BVP_REQUIRE(workspace && workspace_bytes >= L.bytes, BVP_ERR_INVALID,
                "work workspace too small: need %zu bytes", L.bytes);
    cudaStream_t s = as_stream(stream);
    char *ws = static_cast<char *>(workspace);
    auto *cnt = reinterpret_cast<uint4 *>(ws + L.off_cnt);
    auto *part = reinterpret_cast<uint4 *>(ws + L.off_part);
    auto *tot = reinterpret_cast<uint4 *>(ws + L.off_tot);  // n_work, n_partials, n_splits
    auto *tmp = reinterpret_cast<uint4 *>(ws + L.off_tmp);
    auto *keys = reinterpret_cast<uint32_t *>(ws + L.off_keys);
    auto *order = reinterpret_cast<uint32_t *>(ws + L.off_order);
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(n_int_max, 256), 4096));
    work_count_kernel<<<blocks, 256, 0, s>>>(interval_starts, counts, n_int_max, uint32_t(chunk),
                                             cnt);
    device_excl_scan<uint4>(cnt, cnt, n_int_max, part, tot, s);
    // tile < 0: cell order as emitted (per-frame builds: no sort), straight
    // into the work list
    const bool sorted = tile >= 0;
    work_emit_kernel<<<blocks, 256, 0, s>>>(interval_starts, interval_cells, counts,
                                            uint32_t(chunk), cnt,
                                            sorted ? tmp : reinterpret_cast<uint4 *>(work),
                                            sorted ? keys : nullptr,
                                            reinterpret_cast<uint4 *>(splits), ny, tile);
    const int64_t cap = work_cap(n_int_max, n_points, chunk);
    const unsigned cb = static_cast<unsigned>(std::min<int64_t>(ceil_div(cap, 256), 4096));
    const uint32_t *n_work = reinterpret_cast<const uint32_t *>(tot);
    if (!sorted) {
        work_counts_kernel<<<1, 1, 0, s>>>(tot, work_counts);
        return check_launch("make_work");
    }
    work_keys_tail_kernel<<<cb, 256, 0, s>>>(n_work, cap, keys);
    // stable counting sort by length bucket (the association's own sort):
    // longest chunks first, cell order within a bucket, so a warp's groups
    // store to neighbouring cells
    const int rc = bvp_sort_intervals(keys, cap, nkeys, order,
                                      reinterpret_cast<uint32_t *>(ws + L.off_sstarts),
                                      reinterpret_cast<uint32_t *>(ws + L.off_scells),
                                      reinterpret_cast<uint32_t *>(ws + L.off_sfirst), nullptr,
                                      reinterpret_cast<int64_t *>(ws + L.off_scounts),
                                      ws + L.off_sws, L.sort_ws, stream);
    if (rc != BVP_OK) return rc;
    work_gather_kernel<<<cb, 256, 0, s>>>(tmp, order, n_work, reinterpret_cast<uint4 *>(work));
    work_counts_kernel<<<1, 1, 0, s>>>(tot, work_counts);
    return check_launch("make_work");
}

}  // extern "C"

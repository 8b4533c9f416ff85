// partition.cuh -- stable partition of (key, value) pairs by a bounded key,
// from the LSD radix passes of geometry.cu (no per-key global atomics, so it
// suits few distinct keys, e.g. the tiles of the tile plan).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bvp {

// Workspace bytes for up to n_max pairs with keys < 2^key_bits.
size_t stable_partition_ws_bytes(int64_t n_max, int key_bits);

// vals_out[...] = vals[j] for j < *count, ordered by keys[j], ties in input
// order.  Stream ordered, no host sync.
int stable_partition(const uint32_t *keys, const uint32_t *vals, const int64_t *count,
                     int64_t n_max, int key_bits, uint32_t *vals_out, void *ws,
                     size_t ws_bytes, cudaStream_t s);

}  // namespace bvp

// common.cuh -- shared helpers of the sm_100a BEV-pooling kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/bevpool_b200.h"

namespace bvp {

constexpr uint32_t kOOR = BVP_OUT_OF_RANGE;
constexpr int kTileCells = BVP_TILE_CELLS;  // row tile of the backward's grad transpose
constexpr int kUnitCells = 8;               // cells per work unit of the interval kernels

// ---- error channel (host) --------------------------------------------------
void set_error(const char *fmt, ...);
int check_launch(const char *what);

#define BVP_REQUIRE(cond, code, ...)     \
    do {                                 \
        if (!(cond)) {                   \
            ::bvp::set_error(__VA_ARGS__); \
            return (code);               \
        }                                \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Fork / join with this thread's side stream of the current device: work
// launched on `side` is ordered after what was queued on `main` before the
// fork, and `main` waits for it at join() -- by events, so a captured CUDA
// graph gets two parallel branches.
struct SideFork {
    cudaStream_t main, side = nullptr;
    cudaEvent_t fork = nullptr, joined = nullptr;
    // which: one of two side streams (two concurrent forks need distinct ones)
    explicit SideFork(cudaStream_t s, int which = 0) : main(s), side(s) {
        int dev = 0;
        cudaGetDevice(&dev);
        static thread_local cudaStream_t streams[64][2] = {};
        if (dev < 0 || dev >= 64 || which < 0 || which > 1) return;  // run inline
        cudaStream_t &st = streams[dev][which];
        if (!st) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        side = st;
        cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&joined, cudaEventDisableTiming);
        cudaEventRecord(fork, main);
        cudaStreamWaitEvent(side, fork, 0);
    }
    void join() {
        if (side == main) return;
        cudaEventRecord(joined, side);
        cudaStreamWaitEvent(main, joined, 0);
        cudaEventDestroy(fork);
        cudaEventDestroy(joined);
        side = main;
    }
    ~SideFork() { join(); }
};

// ---- device helpers --------------------------------------------------------
__host__ __device__ inline int64_t ceil_div_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// 128-bit read-only load through the non-coherent path.
__device__ __forceinline__ float4 ldg_f4(const float *p) {
    return __ldg(reinterpret_cast<const float4 *>(p));
}
// Streaming 128-bit load (each row used exactly once: do not keep in L1).
__device__ __forceinline__ float4 ldg_stream_f4(const float *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ldg_stream_u4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream_f4(float *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// Read-only loads that ask L2 to fetch the surrounding 256 bytes: strided
// gathers of neighbouring columns by different CTAs then hit L2 instead of
// each pulling its own 32-byte sector from DRAM.
// Read-only loads with a 256-byte L2 prefetch hint, as raw bits, predicated
// in PTX (no branch around each load; 0 when off).  Not volatile: the
// compiler may batch them, and a value is only waited for where it is used
// (the staging loops convert at the store).
__device__ __forceinline__ uint32_t ldg_l2pf_b32(const void *p, bool on) {
    uint32_t r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b32 %0, 0;\n\t"
        "@q ld.global.nc.L2::256B.b32 %0, [%1];\n\t}"
        : "=r"(r)
        : "l"(p), "r"(int(on)));
    return r;
}
__device__ __forceinline__ uint32_t ldg_l2pf_u16(const void *p, bool on) {
    uint16_t r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b16 %0, 0;\n\t"
        "@q ld.global.nc.L2::256B.u16 %0, [%1];\n\t}"
        : "=h"(r)
        : "l"(p), "r"(int(on)));
    return r;
}

__device__ __forceinline__ float bf16_to_f32(uint16_t v) {
    return __uint_as_float(static_cast<uint32_t>(v) << 16);
}

}  // namespace bvp

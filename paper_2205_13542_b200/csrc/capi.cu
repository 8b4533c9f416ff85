// capi.cu -- the C ABI's error channel and version query.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace bvp {

static thread_local char g_last_error[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

// Launch-configuration errors surface synchronously here; asynchronous
// faults surface on the caller's next synchronising call.
int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return BVP_ERR_CUDA;
    }
    return BVP_OK;
}

}  // namespace bvp

extern "C" {

int bvp_abi_version(void) { return BVP_ABI_VERSION; }

const char *bvp_last_error(void) { return bvp::g_last_error; }

}  // extern "C"

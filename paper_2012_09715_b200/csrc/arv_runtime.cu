// Library runtime: per-thread error slot, launch counter, device queries.
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "arv_common.cuh"

namespace arv {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(ARV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return ARV_OK;
}

void note_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }

int device_sm_count() {
    int dev = 0, sms = kNumSMs;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
        return sms;
    return kNumSMs;
}

}  // namespace arv

extern "C" {

int arv_abi_version(void) { return ARV_ABI_VERSION; }
const char *arv_last_error(void) { return arv::g_err; }
uint64_t arv_launch_count(void) { return arv::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"

// Library runtime: per-thread error slot, launch counter, device queries.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <mutex>

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

int resident_ctas(const void *fn, int block, size_t smem) {
    struct Entry {
        const void *fn;
        int block, dev;
        size_t smem;
        int ctas;
    };
    static Entry cache[128];
    static int used = 0;
    static std::mutex mu;
    int dev = 0;
    (void)cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lock(mu);
        for (int i = 0; i < used; ++i)
            if (cache[i].fn == fn && cache[i].block == block && cache[i].smem == smem && cache[i].dev == dev)
                return cache[i].ctas;
    }
    int ctas = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, block, smem) != cudaSuccess || ctas < 1) {
        (void)cudaGetLastError();
        ctas = 1;
    }
    std::lock_guard<std::mutex> lock(mu);
    if (used < 128) cache[used++] = {fn, block, dev, smem, ctas};
    return ctas;
}

}  // namespace arv

extern "C" {

int arv_abi_version(void) { return ARV_ABI_VERSION; }
// sha256 of the csrc/ and include/ sources this library was built from
// (_build.source_hash(), passed as -DARV_SOURCE_HASH): the loader rebuilds or
// refuses a library whose sources changed since (_native._load).
#ifndef ARV_SOURCE_HASH
#define ARV_SOURCE_HASH "unknown"
#endif
// The tagged string is also read from the file itself (no dlopen needed).
static const char kSourceHashTag[] = "ARV_SOURCE_HASH=" ARV_SOURCE_HASH;
const char *arv_source_hash(void) { return kSourceHashTag + 16; }
const char *arv_last_error(void) { return arv::g_err; }
uint64_t arv_launch_count(void) { return arv::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"

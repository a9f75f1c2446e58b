// The reference's calling convention at the plugin boundary: HOST buffers.
//
// approxrv's plugin functions take numpy arrays and fill a caller-allocated
// numpy `out` (_kernels.pyx:16-143, called from sampler.py:91-206 with
// host f64 / f32 batches).  The arv_host_* entry points keep that
// convention for the CUDA plugin: u (and a per-element lambda) are host
// pointers, out is a host pointer, and the call returns when out is written.
//
// Pipeline (one per device, serialised by a mutex; the reference's Cython
// kernels hold the GIL, so one call at a time is the reference's model too):
//
//   host thread            copy-in stream   caller's stream   copy-out stream
//   memcpy u[c] -> pin_in      H2D c          kernel c            D2H c
//   memcpy pin_out -> out[c-S]  ...            ...                 ...
//
// S = 3 slots of pinned + device staging buffers.  Chunk c's host copy into
// pinned memory overlaps the device work of chunks c-1, c-2 and the
// write-back of chunk c-3; the host copies are split over a small thread
// pool (one memcpy thread reaches ~10 GB/s; PCIe 5 x16 moves ~55 GB/s per
// direction).  Every byte of u and out crosses PCIe exactly once and is
// touched by the host exactly once on each side (pageable -> pinned,
// pinned -> pageable): the DMA engines cannot read pageable memory
// asynchronously.
//
// The table arguments are DEVICE pointers (tables are immutable and cached
// on the device by the caller, tables.py:19-24).

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "arv_common.cuh"

namespace arv {
namespace {

// ------------------------------------------------------- memcpy pool --
class CopyPool {
   public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) th_.emplace_back([this] { worker(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    int threads() const { return static_cast<int>(th_.size()) + 1; }

    // memcpy split into parts over the pool and the calling thread.
    void copy(void *dst, const void *src, size_t bytes) {
        constexpr size_t kMinPart = size_t(1) << 20;
        const int parts = static_cast<int>(std::min<size_t>(threads(), (bytes + kMinPart - 1) / kMinPart));
        if (parts <= 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            dst_ = static_cast<char *>(dst);
            src_ = static_cast<const char *>(src);
            bytes_ = bytes;
            part_ = ((bytes + parts - 1) / parts + 4095) & ~size_t(4095);
            nparts_ = parts;
            next_.store(0);
            left_ = parts;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [this] { return left_ == 0; });
    }

   private:
    void work() {
        for (;;) {
            const int p = next_.fetch_add(1);
            if (p >= nparts_) return;
            const size_t lo = std::min(bytes_, static_cast<size_t>(p) * part_);
            const size_t hi = std::min(bytes_, lo + part_);
            if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
            std::lock_guard<std::mutex> lk(m_);
            if (--left_ == 0) done_.notify_one();
        }
    }
    void worker() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    bool stop_ = false;
    uint64_t gen_ = 0;
    char *dst_ = nullptr;
    const char *src_ = nullptr;
    size_t bytes_ = 0, part_ = 0;
    int nparts_ = 0, left_ = 0;
    std::atomic<int> next_{0};
};

int pool_threads() {
    if (const char *e = std::getenv("ARV_HOST_THREADS")) return std::max(1, std::atoi(e));
    // all host threads: the pageable <-> pinned copies are host-memory bound
    // (GPU box, 16 threads: 2 / 4 / 8 / 16 threads -> 145 / 82 / 73 / 61 ms
    // for a 2^28-sample f32 call; 24 threads 62 ms)
    const unsigned hw = std::thread::hardware_concurrency();
    return static_cast<int>(std::max(1u, std::min(32u, hw ? hw : 1u)));
}

// ---------------------------------------------------------- pipeline --
constexpr int kSlots = 3;
constexpr size_t kSlotBytes = size_t(16) << 20;  // per staging buffer
constexpr size_t kMinChunkBytes = size_t(256) << 10;

struct Pipe {
    int dev = -1;
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t ev_up[kSlots], ev_k[kSlots], ev_down[kSlots];
    // buffer b (0 = in0, 1 = in1, 2 = out) of slot s
    void *pin[3][kSlots] = {};
    void *dbuf[3][kSlots] = {};
    double *pin_scalar = nullptr, *d_scalar = nullptr;
    CopyPool *pool = nullptr;
};

std::mutex g_pipe_mu;
Pipe g_pipes[16];

int cuda_fail(cudaError_t e, const char *what) {
    (void)cudaGetLastError();
    return set_error(ARV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
#define ARV_TRY(call)                                               \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);         \
    } while (0)

int pipe_for_device(Pipe *&P) {
    int dev = 0;
    ARV_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 16) return set_error(ARV_ERR_CONFIG, "device index %d out of range", dev);
    P = &g_pipes[dev];
    if (P->dev == dev) return ARV_OK;
    ARV_TRY(cudaStreamCreateWithFlags(&P->up, cudaStreamNonBlocking));
    ARV_TRY(cudaStreamCreateWithFlags(&P->down, cudaStreamNonBlocking));
    for (int s = 0; s < kSlots; ++s) {
        ARV_TRY(cudaEventCreateWithFlags(&P->ev_up[s], cudaEventDisableTiming));
        ARV_TRY(cudaEventCreateWithFlags(&P->ev_k[s], cudaEventDisableTiming));
        ARV_TRY(cudaEventCreateWithFlags(&P->ev_down[s], cudaEventDisableTiming));
    }
    ARV_TRY(cudaHostAlloc(reinterpret_cast<void **>(&P->pin_scalar), 64, cudaHostAllocDefault));
    ARV_TRY(cudaMalloc(reinterpret_cast<void **>(&P->d_scalar), 64));
    P->pool = new CopyPool(pool_threads() - 1);
    P->dev = dev;
    return ARV_OK;
}

int ensure_buffer(Pipe &P, int b) {
    // (write-combined input staging measured slower: 57.7 vs 50.6 ms per
    // 2^28-sample f32 call; registering the caller's arrays in place costs
    // ~28 + 18 ms per GiB to register / unregister, more than the copies)
    for (int s = 0; s < kSlots; ++s) {
        if (!P.pin[b][s]) ARV_TRY(cudaHostAlloc(&P.pin[b][s], kSlotBytes, cudaHostAllocDefault));
        if (!P.dbuf[b][s]) ARV_TRY(cudaMalloc(&P.dbuf[b][s], kSlotBytes));
    }
    return ARV_OK;
}

// One elementwise op over host arrays.  in1 may be null; es_* are element
// sizes in bytes; launch(d_in0, d_in1, d_out, count, stream) enqueues the
// device kernel for one chunk.
// `scalar` (optional) is copied to a device double on the caller's stream
// before the first chunk; launch receives its device address.
template <class Launch>
int host_pipeline(const void *in0, size_t es0, const void *in1, size_t es1, void *out, size_t es_out, int64_t n,
                  cudaStream_t s, const char *what, Launch launch, const double *scalar = nullptr) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "%s: negative length", what);
    if (n == 0) return ARV_OK;
    if (!in0 || !out || (es1 && !in1)) return set_error(ARV_ERR_CONFIG, "%s: null host pointer", what);
    std::lock_guard<std::mutex> lock(g_pipe_mu);
    Pipe *P = nullptr;
    if (int rc = pipe_for_device(P)) return rc;
    if (int rc = ensure_buffer(*P, 0)) return rc;
    if (in1)
        if (int rc = ensure_buffer(*P, 1)) return rc;
    if (int rc = ensure_buffer(*P, 2)) return rc;
    const double *d_scalar = nullptr;
    if (scalar) {
        // the previous call on this pipe has completed (every call drains),
        // so the pinned scalar is free
        *P->pin_scalar = *scalar;
        ARV_TRY(cudaMemcpyAsync(P->d_scalar, P->pin_scalar, sizeof(double), cudaMemcpyHostToDevice, s));
        d_scalar = P->d_scalar;
    }
    const size_t es_max = std::max({es0, in1 ? es1 : size_t(0), es_out});
    const int64_t cap = static_cast<int64_t>(kSlotBytes / es_max);
    // chunks small enough that a mid-sized call still pipelines (>= ~8 chunks)
    const int64_t want = static_cast<int64_t>(std::max(kMinChunkBytes / es_max, size_t(1)));
    const int64_t chunk = std::min(cap, std::max(want, (n + 7) / 8));
    const int64_t nchunks = (n + chunk - 1) / chunk;
    const char *src0 = static_cast<const char *>(in0);
    const char *src1 = static_cast<const char *>(in1);
    char *dst = static_cast<char *>(out);
    auto drain = [&](int64_t c) -> int {  // chunk c's result -> caller's out
        const int slot = static_cast<int>(c % kSlots);
        const int64_t lo = c * chunk, cnt = std::min(chunk, n - lo);
        ARV_TRY(cudaEventSynchronize(P->ev_down[slot]));
        P->pool->copy(dst + lo * es_out, P->pin[2][slot], static_cast<size_t>(cnt) * es_out);
        return ARV_OK;
    };
    for (int64_t c = 0; c < nchunks; ++c) {
        const int slot = static_cast<int>(c % kSlots);
        if (c >= kSlots)  // frees the slot: its D2H (hence its kernel and H2D) is complete
            if (int rc = drain(c - kSlots)) return rc;
        const int64_t lo = c * chunk, cnt = std::min(chunk, n - lo);
        P->pool->copy(P->pin[0][slot], src0 + lo * es0, static_cast<size_t>(cnt) * es0);
        ARV_TRY(cudaMemcpyAsync(P->dbuf[0][slot], P->pin[0][slot], cnt * es0, cudaMemcpyHostToDevice, P->up));
        if (in1) {
            P->pool->copy(P->pin[1][slot], src1 + lo * es1, static_cast<size_t>(cnt) * es1);
            ARV_TRY(cudaMemcpyAsync(P->dbuf[1][slot], P->pin[1][slot], cnt * es1, cudaMemcpyHostToDevice, P->up));
        }
        ARV_TRY(cudaEventRecord(P->ev_up[slot], P->up));
        ARV_TRY(cudaStreamWaitEvent(s, P->ev_up[slot], 0));
        if (int rc = launch(P->dbuf[0][slot], in1 ? P->dbuf[1][slot] : d_scalar, P->dbuf[2][slot], cnt, s))
            return rc;
        ARV_TRY(cudaEventRecord(P->ev_k[slot], s));
        ARV_TRY(cudaStreamWaitEvent(P->down, P->ev_k[slot], 0));
        ARV_TRY(cudaMemcpyAsync(P->pin[2][slot], P->dbuf[2][slot], cnt * es_out, cudaMemcpyDeviceToHost, P->down));
        ARV_TRY(cudaEventRecord(P->ev_down[slot], P->down));
    }
    for (int64_t c = std::max<int64_t>(0, nchunks - kSlots); c < nchunks; ++c)
        if (int rc = drain(c)) return rc;
    return ARV_OK;
}

}  // namespace
}  // namespace arv

using namespace arv;

extern "C" {

int arv_host_constant_eval(const double *values, int64_t nvals, const double *u, double *out, int64_t n, void *stream) {
    return host_pipeline(u, 8, nullptr, 0, out, 8, n, as_stream(stream), "arv_host_constant_eval",
                         [&](const void *a, const void *, void *o, int64_t cnt, cudaStream_t s) {
                             return arv_constant_eval(values, nvals, static_cast<const double *>(a),
                                                      static_cast<double *>(o), cnt, s);
                         });
}

int arv_host_dyadic_index(const double *u, int64_t n, int64_t cap, int64_t *out, void *stream) {
    return host_pipeline(u, 8, nullptr, 0, out, 8, n, as_stream(stream), "arv_host_dyadic_index",
                         [&](const void *a, const void *, void *o, int64_t cnt, cudaStream_t s) {
                             return arv_dyadic_index(static_cast<const double *>(a), cnt, cap,
                                                     static_cast<int64_t *>(o), s);
                         });
}

int arv_host_dyadic_index32(const float *u, int64_t n, int64_t cap, int64_t *out, void *stream) {
    return host_pipeline(u, 4, nullptr, 0, out, 8, n, as_stream(stream), "arv_host_dyadic_index32",
                         [&](const void *a, const void *, void *o, int64_t cnt, cudaStream_t s) {
                             return arv_dyadic_index32(static_cast<const float *>(a), cnt, cap,
                                                       static_cast<int64_t *>(o), s);
                         });
}

int arv_host_dyadic_eval(const double *coeffs, int degree, int64_t K1, const double *u, double *out, int64_t n,
                         void *stream) {
    return host_pipeline(u, 8, nullptr, 0, out, 8, n, as_stream(stream), "arv_host_dyadic_eval",
                         [&](const void *a, const void *, void *o, int64_t cnt, cudaStream_t s) {
                             return arv_dyadic_eval(coeffs, degree, K1, static_cast<const double *>(a),
                                                    static_cast<double *>(o), cnt, s);
                         });
}

int arv_host_dyadic_eval32(const float *coeffs, int degree, int64_t K1, const float *u, float *out, int64_t n,
                           void *stream) {
    return host_pipeline(u, 4, nullptr, 0, out, 4, n, as_stream(stream), "arv_host_dyadic_eval32",
                         [&](const void *a, const void *, void *o, int64_t cnt, cudaStream_t s) {
                             return arv_dyadic_eval32(coeffs, degree, K1, static_cast<const float *>(a),
                                                      static_cast<float *>(o), cnt, s);
                         });
}

int arv_host_subdyadic_eval32(const float *coeffs, int degree, int K, int sub_bits, const float *u, float *out,
                              int64_t n, void *stream) {
    return host_pipeline(u, 4, nullptr, 0, out, 4, n, as_stream(stream), "arv_host_subdyadic_eval32",
                         [&](const void *a, const void *, void *o, int64_t cnt, cudaStream_t s) {
                             return arv_subdyadic_eval32(coeffs, degree, K, sub_bits, static_cast<const float *>(a),
                                                         static_cast<float *>(o), cnt, s);
                         });
}

int arv_host_ncchi2_eval(const double *stacks, int64_t n_knots, int degree, int64_t K1, double nu, const double *u,
                         const double *lam, int64_t nlam, double *out, int64_t n, void *stream) {
    if (nlam != 1 && nlam != n)
        return set_error(ARV_ERR_CONFIG, "arv_host_ncchi2_eval: lam must have 1 or n elements");
    if (!lam) return set_error(ARV_ERR_CONFIG, "arv_host_ncchi2_eval: null lam");
    if (nlam == 1)  // shared lambda: one device scalar, read by every chunk's kernel
        return host_pipeline(
            u, 8, nullptr, 0, out, 8, n, as_stream(stream), "arv_host_ncchi2_eval",
            [&](const void *a, const void *l, void *o, int64_t cnt, cudaStream_t s) {
                return arv_ncchi2_eval(stacks, n_knots, degree, K1, nu, static_cast<const double *>(a),
                                       static_cast<const double *>(l), 1, static_cast<double *>(o), cnt, s);
            },
            lam);
    return host_pipeline(u, 8, lam, 8, out, 8, n, as_stream(stream), "arv_host_ncchi2_eval",
                         [&](const void *a, const void *l, void *o, int64_t cnt, cudaStream_t s) {
                             return arv_ncchi2_eval(stacks, n_knots, degree, K1, nu, static_cast<const double *>(a),
                                                    static_cast<const double *>(l), cnt, static_cast<double *>(o),
                                                    cnt, s);
                         });
}

int arv_host_gaussian_inv_cdf(const double *u, double *out, int64_t n, void *stream) {
    return host_pipeline(u, 8, nullptr, 0, out, 8, n, as_stream(stream), "arv_host_gaussian_inv_cdf",
                         [&](const void *a, const void *, void *o, int64_t cnt, cudaStream_t s) {
                             return arv_gaussian_inv_cdf(static_cast<const double *>(a), static_cast<double *>(o),
                                                         cnt, s);
                         });
}

}  // extern "C"

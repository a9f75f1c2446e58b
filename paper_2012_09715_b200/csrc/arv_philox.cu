// Philox-4x64-10 replay generator: the reference's own uniform stream
// (UniformStream, sampler.py:26-66) on the device, bit-exact with
// numpy.random.Philox, fused with the reference evaluators so that
// `evaluate(table, UniformStream(seed, sid, counter).uniforms(n))` is
// reproduced without materialising the uniforms.  One thread per Philox
// block (4 words); the counter may start mid-block.
#include "arv_common.cuh"
#include "arv_eval_dev.cuh"

namespace arv {

constexpr int kPhBlock = 256;

struct PhArgs {
    uint64_t seed, sid, first;  // first word index
    int64_t n;
};

template <class F>
__device__ __forceinline__ void philox_loop(const PhArgs &a, const F &emit) {
    const uint64_t b0 = a.first >> 2;
    const uint64_t b1 = (a.first + static_cast<uint64_t>(a.n) - 1) >> 2;
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t b = b0 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b <= b1; b += T) {
        const uint64_t c = b + 1;
        const Philox4 r = philox4x64_10(c, c == 0 ? 1u : 0u, 0, 0, a.seed, a.sid);
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const uint64_t w = 4 * b + l;
            if (w >= a.first && w < a.first + static_cast<uint64_t>(a.n)) emit(w - a.first, r.w[l]);
        }
    }
}

__global__ void __launch_bounds__(kPhBlock) k_philox_words(PhArgs a, uint64_t *__restrict__ out) {
    philox_loop(a, [&](uint64_t i, uint64_t w) { out[i] = w; });
}

// kind 0: uniform; 1: constant_eval (_kernels.pyx:16-23); 2: dyadic_eval
// (_kernels.pyx:56-73); 3: AS241 gaussian_inv_cdf (exact_dist.py:87-126).
template <int KIND, int DEG>
__global__ void __launch_bounds__(kPhBlock) k_philox_eval(PhArgs a, const double *__restrict__ tab, int64_t tab_n,
                                                          double *__restrict__ out) {
    extern __shared__ double smd[];
    if constexpr (KIND == 1 || KIND == 2) {
        for (int64_t i = threadIdx.x; i < tab_n; i += blockDim.x) smd[i] = __ldg(tab + i);
        __syncthreads();
    }
    philox_loop(a, [&](uint64_t i, uint64_t w) {
        const double u = u64_to_f64(w);
        double r;
        if constexpr (KIND == 0) {
            r = u;
        } else if constexpr (KIND == 1) {
            long long idx = static_cast<long long>(__dmul_rn(static_cast<double>(tab_n), u));
            idx = idx < tab_n ? idx : tab_n - 1;
            r = smd[idx];
        } else if constexpr (KIND == 2) {
            r = dyadic_eval1<DEG>(smd, tab_n / (DEG + 1), u);
        } else {
            r = as241_f64(u);
        }
        __stcs(out + i, r);
    });
}

static int ph_grid(int64_t n) { return stream_grid(n / 4 + 2, kPhBlock, 8); }

}  // namespace arv

using namespace arv;

extern "C" {

int arv_philox_words(uint64_t seed, uint64_t stream_id, uint64_t counter, uint64_t *out, int64_t n, void *stream) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "cannot draw a negative number of words");
    if (n == 0) return ARV_OK;
    k_philox_words<<<ph_grid(n), kPhBlock, 0, as_stream(stream)>>>(PhArgs{seed, stream_id, counter, n}, out);
    note_launch();
    return check_launch("arv_philox_words");
}

int arv_philox_eval_f64(uint64_t seed, uint64_t stream_id, uint64_t counter, int kind, const double *table,
                        int degree, int64_t table_cols, double *out, int64_t n, void *stream) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "cannot draw a negative number of words");
    if (kind < 0 || kind > 3) return set_error(ARV_ERR_CONFIG, "unknown philox evaluation kind %d", kind);
    if (n == 0) return ARV_OK;
    const PhArgs a{seed, stream_id, counter, n};
    const int grid = ph_grid(n);
    cudaStream_t s = as_stream(stream);
    if (kind == 0) {
        k_philox_eval<0, 1><<<grid, kPhBlock, 0, s>>>(a, nullptr, 0, out);
    } else if (kind == 3) {
        k_philox_eval<3, 1><<<grid, kPhBlock, 0, s>>>(a, nullptr, 0, out);
    } else if (kind == 1) {
        if (table_cols < 1 || table_cols > 8192) return set_error(ARV_ERR_CONFIG, "constant table size out of range");
        k_philox_eval<1, 1><<<grid, kPhBlock, sizeof(double) * table_cols, s>>>(a, table, table_cols, out);
    } else {
        if (table_cols < 2 || table_cols > 4096) return set_error(ARV_ERR_CONFIG, "bad table interval count");
        const int64_t tn = (degree + 1) * table_cols;
        const size_t smem = sizeof(double) * tn;
        switch (degree) {
            case 1: k_philox_eval<2, 1><<<grid, kPhBlock, smem, s>>>(a, table, tn, out); break;
            case 2: k_philox_eval<2, 2><<<grid, kPhBlock, smem, s>>>(a, table, tn, out); break;
            case 3: k_philox_eval<2, 3><<<grid, kPhBlock, smem, s>>>(a, table, tn, out); break;
            case 4: k_philox_eval<2, 4><<<grid, kPhBlock, smem, s>>>(a, table, tn, out); break;
            case 5: k_philox_eval<2, 5><<<grid, kPhBlock, smem, s>>>(a, table, tn, out); break;
            default: return set_error(ARV_ERR_CONFIG, "polynomial degree must be in [1, 5], got %d", degree);
        }
    }
    note_launch();
    return check_launch("arv_philox_eval_f64");
}

}  // extern "C"

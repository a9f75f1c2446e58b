// Philox-4x64-10 replay generator: the reference's own uniform stream
// (UniformStream, sampler.py:26-66) on the device, bit-exact with
// numpy.random.Philox, fused with the reference evaluators so that
// `evaluate(table, UniformStream(seed, sid, counter).uniforms(n))` is
// reproduced without materialising the uniforms.  One thread per Philox
// block (4 words); the counter may start mid-block.
#include "arv_common.cuh"
#include "arv_eval_dev.cuh"

#include <cstring>
#include <type_traits>

namespace arv {

constexpr int kPhBlock = 256;

struct PhArgs {
    uint64_t seed, sid, first;  // first word index
    int64_t n;
};

// Each thread takes two consecutive Philox blocks per iteration (two
// independent 10-round chains in flight); blocks entirely inside the call's
// word range go through emit4 (vector stores when `vec`), the at most two
// partial blocks at the ends through emit1.
template <class F4, class F1>
__device__ __forceinline__ void philox_loop(const PhArgs &a, bool vec, const F4 &emit4, const F1 &emit1) {
    const uint64_t first = a.first, end = a.first + static_cast<uint64_t>(a.n);
    const uint64_t b0 = first >> 2, nb = ((end - 1) >> 2) - b0 + 1;
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    auto block = [&](uint64_t b, const Philox4 &r) {
        if (4 * b >= first && 4 * b + 4 <= end) {
            emit4(4 * b - first, r, vec);
        } else {
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const uint64_t w = 4 * b + l;
                if (w >= first && w < end) emit1(w - first, r.w[l]);
            }
        }
    };
    for (uint64_t k = 2 * (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x); k < nb; k += 2 * T) {
        const uint64_t b = b0 + k;
        const uint64_t c0 = b + 1, c1 = b + 2;  // numpy pre-increments the counter
        const Philox4 r0 = philox4x64_10(c0, c0 == 0 ? 1u : 0u, 0, 0, a.seed, a.sid);
        const Philox4 r1 = philox4x64_10(c1, c1 == 0 ? 1u : 0u, 0, 0, a.seed, a.sid);
        block(b, r0);
        if (k + 1 < nb) block(b + 1, r1);
    }
}

// Four results of one block at out[i0 .. i0 + 3]: two 16-byte streaming stores
// when the call is 4-word aligned, else four scalar ones.
template <class T>
__device__ __forceinline__ void store4(T *out, uint64_t i0, const T (&v)[4], bool vec) {
    if (vec) {
        using V2 = typename std::conditional<sizeof(T) == 8, ulonglong2, uint2>::type;
        V2 *o = reinterpret_cast<V2 *>(out + i0);
        V2 x, y;
        memcpy(&x, &v[0], sizeof(V2));
        memcpy(&y, &v[2], sizeof(V2));
        __stcs(o, x);
        __stcs(o + 1, y);
    } else {
#pragma unroll
        for (int l = 0; l < 4; ++l) __stcs(out + i0 + l, v[l]);
    }
}

__global__ void __launch_bounds__(kPhBlock) k_philox_words(PhArgs a, bool vec, uint64_t *__restrict__ out) {
    philox_loop(
        a, vec, [&](uint64_t i0, const Philox4 &r, bool v) { store4(out, i0, r.w, v); },
        [&](uint64_t i, uint64_t w) { out[i] = w; });
}

// kind 0: uniform; 1: constant_eval (_kernels.pyx:16-23); 2: dyadic_eval
// (_kernels.pyx:56-73); 3: AS241 gaussian_inv_cdf (exact_dist.py:87-126).
template <int KIND, int DEG>
__device__ __forceinline__ double philox_map(const double *smd, int64_t tab_n, double u) {
    if constexpr (KIND == 0) {
        return u;
    } else if constexpr (KIND == 1) {
        long long idx = static_cast<long long>(__dmul_rn(static_cast<double>(tab_n), u));
        idx = idx < tab_n ? idx : tab_n - 1;
        return smd[idx];
    } else if constexpr (KIND == 2) {
        return dyadic_eval1<DEG>(smd, tab_n / (DEG + 1), u);
    } else {
        return as241_f64(u);
    }
}

template <int KIND, int DEG>
__global__ void __launch_bounds__(kPhBlock) k_philox_eval(PhArgs a, bool vec, const double *__restrict__ tab,
                                                          int64_t tab_n, double *__restrict__ out) {
    extern __shared__ double smd[];
    if constexpr (KIND == 1 || KIND == 2) {
        for (int64_t i = threadIdx.x; i < tab_n; i += blockDim.x) smd[i] = __ldg(tab + i);
        __syncthreads();
    }
    philox_loop(
        a, vec,
        [&](uint64_t i0, const Philox4 &r, bool v) {
            double u[4], z[4];
#pragma unroll
            for (int l = 0; l < 4; ++l) u[l] = u64_to_f64(r.w[l]);
            if constexpr (KIND == 3) {
                as241_f64_batch<4>(u, z);  // tail log/sqrt compacted over the 4 per lane
            } else {
#pragma unroll
                for (int l = 0; l < 4; ++l) z[l] = philox_map<KIND, DEG>(smd, tab_n, u[l]);
            }
            store4(out, i0, z, v);
        },
        [&](uint64_t i, uint64_t w) { __stcs(out + i, philox_map<KIND, DEG>(smd, tab_n, u64_to_f64(w))); });
}

static int ph_grid(int64_t n) { return stream_grid(n / 8 + 2, kPhBlock, 8); }
// 16-byte stores need a 4-word-aligned counter and a 16-byte-aligned output
static bool ph_vec(uint64_t counter, const void *out) {
    return (counter & 3u) == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
}

}  // namespace arv

using namespace arv;

extern "C" {

int arv_philox_words(uint64_t seed, uint64_t stream_id, uint64_t counter, uint64_t *out, int64_t n, void *stream) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "cannot draw a negative number of words");
    if (n == 0) return ARV_OK;
    k_philox_words<<<ph_grid(n), kPhBlock, 0, as_stream(stream)>>>(PhArgs{seed, stream_id, counter, n},
                                                                    ph_vec(counter, out), out);
    note_launch();
    return check_launch("arv_philox_words");
}

int arv_philox_eval_f64(uint64_t seed, uint64_t stream_id, uint64_t counter, int kind, const double *table,
                        int degree, int64_t table_cols, double *out, int64_t n, void *stream) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "cannot draw a negative number of words");
    if (kind < 0 || kind > 3) return set_error(ARV_ERR_CONFIG, "unknown philox evaluation kind %d", kind);
    if (n == 0) return ARV_OK;
    const PhArgs a{seed, stream_id, counter, n};
    const bool vec = ph_vec(counter, out);
    const int grid = ph_grid(n);
    cudaStream_t s = as_stream(stream);
    if (kind == 0) {
        k_philox_eval<0, 1><<<grid, kPhBlock, 0, s>>>(a, vec, nullptr, 0, out);
    } else if (kind == 3) {
        k_philox_eval<3, 1><<<grid, kPhBlock, 0, s>>>(a, vec, nullptr, 0, out);
    } else if (kind == 1) {
        if (table_cols < 1 || table_cols > 8192) return set_error(ARV_ERR_CONFIG, "constant table size out of range");
        k_philox_eval<1, 1><<<grid, kPhBlock, sizeof(double) * table_cols, s>>>(a, vec, table, table_cols, out);
    } else {
        if (table_cols < 2 || table_cols > 4096) return set_error(ARV_ERR_CONFIG, "bad table interval count");
        const int64_t tn = (degree + 1) * table_cols;
        const size_t smem = sizeof(double) * tn;
        switch (degree) {
            case 1: k_philox_eval<2, 1><<<grid, kPhBlock, smem, s>>>(a, vec, table, tn, out); break;
            case 2: k_philox_eval<2, 2><<<grid, kPhBlock, smem, s>>>(a, vec, table, tn, out); break;
            case 3: k_philox_eval<2, 3><<<grid, kPhBlock, smem, s>>>(a, vec, table, tn, out); break;
            case 4: k_philox_eval<2, 4><<<grid, kPhBlock, smem, s>>>(a, vec, table, tn, out); break;
            case 5: k_philox_eval<2, 5><<<grid, kPhBlock, smem, s>>>(a, vec, table, tn, out); break;
            default: return set_error(ARV_ERR_CONFIG, "polynomial degree must be in [1, 5], got %d", degree);
        }
    }
    note_launch();
    return check_launch("arv_philox_eval_f64");
}

}  // extern "C"

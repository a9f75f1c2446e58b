// Drop-in replacements of the reference kernel plugin (_kernels.pyx:16-143)
// on device arrays, plus the f32 octave x sub-interval evaluator and the
// AS241 exact quantile.  Element-wise, HBM-bound: tables are staged once per
// CTA in shared memory, inputs are read once and outputs written once.
#include "arv_common.cuh"
#include "arv_eval_dev.cuh"


namespace arv {

constexpr int kEvalBlock = 256;
constexpr int kEvalPerSM = 8;

// Grid = resident CTAs per SM (from the occupancy calculator, cached per
// kernel and dynamic smem size) x SMs, so the grid-stride loop runs as one
// wave whatever the kernel's register count; small n gets fewer CTAs.
static int eval_grid(const void *fn, int64_t n, size_t smem) {
    const int per_sm = resident_ctas(fn, kEvalBlock, smem);
    return stream_grid(n, kEvalBlock, per_sm < kEvalPerSM ? per_sm : kEvalPerSM);
}


// Element-wise map out[i] = f(u[i] [, aux[i]]).  When every pointer is
// 16-byte aligned the body moves 16-byte vectors, two per thread in flight
// (a scalar 4-byte stream keeps ~1 MB in flight chip-wide, far below the
// ~6 MB the HBM latency-bandwidth product asks for); the remainder and
// misaligned views take the scalar grid-stride loop.  Streaming cache hints
// on both sides: every byte is touched once.
template <typename In, typename Out, int V, typename F, typename... A>
__device__ __forceinline__ void ew_apply(const uint4 &r, const uint4 *ra, Out *dst, F &f) {
    In a[V];
    memcpy(a, &r, 16);
    Out b[V];
    if constexpr (sizeof...(A) == 0) {
#pragma unroll
        for (int k = 0; k < V; ++k) b[k] = f(a[k]);
    } else {
        In x[V];
        memcpy(x, ra, 16);
#pragma unroll
        for (int k = 0; k < V; ++k) b[k] = f(a[k], x[k]);
    }
    constexpr int VO = static_cast<int>(sizeof(b) / 16);
#pragma unroll
    for (int k = 0; k < VO; ++k) {
        uint4 w;
        memcpy(&w, reinterpret_cast<const char *>(b) + 16 * k, 16);
        __stcs(reinterpret_cast<uint4 *>(dst) + k, w);
    }
}

template <bool AUX, typename In, typename Out, typename F>
__device__ __forceinline__ void ew_map(const In *__restrict__ u, const In *__restrict__ aux, Out *__restrict__ out,
                                       int64_t n, F f) {
    constexpr int V = 16 / sizeof(In);
    static_assert(sizeof(Out) >= sizeof(In), "output vectors are whole 16-byte stores");
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    uintptr_t align = reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(out);
    if (AUX) align |= reinterpret_cast<uintptr_t>(aux);
    int64_t head = 0;
    if ((align & 15) == 0) {
        const int64_t nv = n / V;
        const uint4 *uv = reinterpret_cast<const uint4 *>(u);
        const uint4 *xv = reinterpret_cast<const uint4 *>(aux);
        for (int64_t i = tid; i < nv; i += 2 * stride) {
            const bool two = i + stride < nv;
            const uint4 ra = __ldcs(uv + i);
            uint4 rb = ra, xa, xb;
            if (two) rb = __ldcs(uv + i + stride);
            if (AUX) {
                xa = __ldcs(xv + i);
                xb = two ? __ldcs(xv + i + stride) : xa;
            }
            if constexpr (AUX) {
                ew_apply<In, Out, V, F, In>(ra, &xa, out + i * V, f);
                if (two) ew_apply<In, Out, V, F, In>(rb, &xb, out + (i + stride) * V, f);
            } else {
                ew_apply<In, Out, V, F>(ra, nullptr, out + i * V, f);
                if (two) ew_apply<In, Out, V, F>(rb, nullptr, out + (i + stride) * V, f);
            }
        }
        head = nv * V;
    }
    for (int64_t i = head + tid; i < n; i += stride) {
        if constexpr (AUX) __stcs(out + i, f(__ldcs(u + i), __ldcs(aux + i)));
        else __stcs(out + i, f(__ldcs(u + i)));
    }
}

// ------------------------------------------------------- constant_eval --
// _kernels.pyx:16-23: idx = (long long)(nvals * u), idx = min(idx, nvals-1).
__global__ void __launch_bounds__(kEvalBlock, 6) k_constant_eval(const double *__restrict__ values, int64_t nvals,
                                                              int use_smem, const double *__restrict__ u,
                                                              double *__restrict__ out, int64_t n) {
    extern __shared__ double smd[];
    const double scale = static_cast<double>(nvals);
    auto index = [=](double ui) {
        long long idx = static_cast<long long>(__dmul_rn(scale, ui));
        idx = idx < nvals ? idx : nvals - 1;
        return idx < 0 ? 0 : idx;  // memory-safety clamp (u outside the (0,1) contract)
    };
    if (use_smem) {  // separate bodies so the staged table is read with LDS, not generic loads
        for (int i = threadIdx.x; i < nvals; i += blockDim.x) smd[i] = __ldg(values + i);
        __syncthreads();
        ew_map<false>(u, u, out, n, [=](double ui) { return smd[index(ui)]; });
    } else {
        ew_map<false>(u, u, out, n, [=](double ui) { return __ldg(values + index(ui)); });
    }
}

// -------------------------------------------------------- dyadic_index --
__global__ void __launch_bounds__(kEvalBlock, kEvalPerSM) k_dyadic_index(const double *__restrict__ u, int64_t cap,
                                                             long long *__restrict__ out, int64_t n) {
    ew_map<false>(u, u, out, n, [=](double ui) { return dyadic_idx64(ui, cap); });
}
__global__ void __launch_bounds__(kEvalBlock) k_dyadic_index32(const float *__restrict__ u, int64_t cap,
                                                               long long *__restrict__ out, int64_t n) {
    ew_map<false>(u, u, out, n, [=](float ui) { return dyadic_idx32(ui, cap); });
}

// --------------------------------------------------------- dyadic_eval --
// _kernels.pyx:56-73 (f64) and :76-93 (f32).  coeffs (degree+1, K1) staged
// in shared memory; Horner with separately rounded mul/add.
template <int DEG>
__global__ void __launch_bounds__(kEvalBlock) k_dyadic_eval(const double *__restrict__ coeffs, int64_t K1,
                                                            const double *__restrict__ u, double *__restrict__ out,
                                                            int64_t n) {
    extern __shared__ double smd[];
    for (int i = threadIdx.x; i < (DEG + 1) * K1; i += blockDim.x) smd[i] = __ldg(coeffs + i);
    __syncthreads();
    const long long cap = K1 - 1;
    ew_map<false>(u, u, out, n, [=](double ui) {
        const bool pred = ui < 0.5;
        const double v = pred ? ui : __dsub_rn(1.0, ui);
        long long idx = dyadic_idx64(v, cap);
        idx = idx < 0 ? 0 : idx;
        double z = smd[DEG * K1 + idx];
#pragma unroll
        for (int d = DEG - 1; d >= 0; --d) z = __dadd_rn(__dmul_rn(z, v), smd[d * K1 + idx]);
        return pred ? z : -z;
    });
}

template <int DEG>
__global__ void __launch_bounds__(kEvalBlock) k_dyadic_eval32(const float *__restrict__ coeffs, int64_t K1,
                                                              const float *__restrict__ u, float *__restrict__ out,
                                                              int64_t n) {
    extern __shared__ float smf[];
    for (int i = threadIdx.x; i < (DEG + 1) * K1; i += blockDim.x) smf[i] = __ldg(coeffs + i);
    __syncthreads();
    const long long cap = K1 - 1;
    ew_map<false>(u, u, out, n, [=](float ui) {
        const bool pred = ui < 0.5f;
        const float v = pred ? ui : __fsub_rn(1.0f, ui);
        long long idx = dyadic_idx32(v, cap);
        idx = idx < 0 ? 0 : idx;
        float z = smf[DEG * K1 + idx];
#pragma unroll
        for (int d = DEG - 1; d >= 0; --d) z = __fadd_rn(__fmul_rn(z, v), smf[d * K1 + idx]);
        return pred ? z : -z;
    });
}

// --------------------------------------------- octave x sub-interval f32 --
template <int DEG>
__global__ void __launch_bounds__(kEvalBlock) k_subdyadic_eval32(const float *__restrict__ coeffs, int K, int b,
                                                                 const float *__restrict__ u, float *__restrict__ out,
                                                                 int64_t n) {
    extern __shared__ float smf[];
    const int nsub = 1 << b;
    const int plane = (K + 1) << b;
    for (int e = threadIdx.x; e < plane; e += blockDim.x) {
        const int r = e >> b, s = e & (nsub - 1);
        const int j = K - r;
        for (int d = 0; d <= DEG; ++d)
            smf[d * plane + e] =
                j == 0 ? 0.0f : __ldg(coeffs + (static_cast<int64_t>(d) * K + (j - 1)) * nsub + (j == K ? 0 : s));
    }
    __syncthreads();
    const int shift = 23 - b, base = (126 - K) << b;
    ew_map<false>(u, u, out, n, [=](float ui) {
        const bool pred = ui < 0.5f;
        const float v = pred ? ui : __fsub_rn(1.0f, ui);
        int e = static_cast<int>(__float_as_uint(v) >> shift) - base;
        e = min(max(e, 0), plane - 1);
        float z = smf[DEG * plane + e];
#pragma unroll
        for (int d = DEG - 1; d >= 0; --d) z = __fadd_rn(__fmul_rn(z, v), smf[d * plane + e]);
        return pred ? z : -z;
    });
}

// --------------------------------------------------------- ncchi2_eval --
// _kernels.pyx:96-143.  stacks (2, n_knots, DEG+1, K1): upper half at 0,
// lower at 1; knot bracketing j = min(floor(sqrt(nu/(lam+nu)) (n_knots-1)),
// n_knots-2), linear interpolation in t.  All IEEE (div/sqrt round-to-nearest).
template <int DEG>
__device__ __forceinline__ void ncchi2_map(const double *tab, int64_t n_knots, int64_t K1, double nu,
                                           const double *__restrict__ u, const double *__restrict__ lam, int64_t nlam,
                                           double *__restrict__ out, int64_t n) {
    if (nlam == 1) {  // shared lambda: knot bracket (two sqrt, one div) once per thread
        const NcKnot kn = ncchi2_knot(n_knots, nu, __ldg(lam));
        ew_map<false>(u, u, out, n, [=](double ui) { return ncchi2_eval_at<DEG>(tab, n_knots, K1, kn, ui); });
    } else {
        ew_map<true>(u, lam, out, n, [=](double ui, double li) {
            return ncchi2_eval_at<DEG>(tab, n_knots, K1, ncchi2_knot(n_knots, nu, li), ui);
        });
    }
}

template <int DEG>
// Linear tables (the shipped ones): 64 registers, 4 CTAs/SM (20 B spill) --
// more bytes in flight: shared-lambda 0.96 -> 0.87 ms at 2^28.  Higher
// degrees keep the ~80-register, 3-CTA shape.
__global__ void __launch_bounds__(kEvalBlock, DEG == 1 ? 4 : 3) k_ncchi2_eval(const double *__restrict__ stacks, int64_t n_knots,
                                                            int64_t K1, int use_smem, double nu,
                                                            const double *__restrict__ u,
                                                            const double *__restrict__ lam, int64_t nlam,
                                                            double *__restrict__ out, int64_t n) {
    extern __shared__ double smd[];
    if (use_smem) {
        const int64_t total = 2 * n_knots * (DEG + 1) * K1;
        for (int64_t i = threadIdx.x; i < total; i += blockDim.x) smd[i] = __ldg(stacks + i);
        __syncthreads();
        ncchi2_map<DEG>(smd, n_knots, K1, nu, u, lam, nlam, out, n);
    } else {
        ncchi2_map<DEG>(stacks, n_knots, K1, nu, u, lam, nlam, out, n);
    }
}

// ---------------------------------------------------------- AS241 exact --
// Four elements per thread and pass (two 16-byte vectors) so that the tail's
// log / sqrt is compacted 4-wide across the warp (as241_f64_batch).
__global__ void __launch_bounds__(kEvalBlock) k_gauss_inv_cdf(const double *__restrict__ u, double *__restrict__ out,
                                                              int64_t n) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int64_t head = 0;
    if (((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
        const int64_t nq = n / 4;  // groups of 4 doubles
        const double2 *uv = reinterpret_cast<const double2 *>(u);
        double2 *ov = reinterpret_cast<double2 *>(out);
        for (int64_t i = tid; i < nq; i += stride) {
            const double2 a = __ldcs(uv + 2 * i), b = __ldcs(uv + 2 * i + 1);
            const double x[4] = {a.x, a.y, b.x, b.y};
            double r[4];
            as241_f64_batch<4>(x, r);
            __stcs(ov + 2 * i, make_double2(r[0], r[1]));
            __stcs(ov + 2 * i + 1, make_double2(r[2], r[3]));
        }
        head = nq * 4;
    }
    for (int64_t i = head + tid; i < n; i += stride) __stcs(out + i, as241_f64(__ldcs(u + i)));
}
__global__ void __launch_bounds__(kEvalBlock) k_gauss_inv_cdf32(const float *__restrict__ u, float *__restrict__ out,
                                                                int64_t n) {
    ew_map<false>(u, u, out, n, [](float ui) { return as241_f32(ui); });
}

static int finish(const char *what) {
    note_launch();
    return check_launch(what);
}

static int set_smem(const void *fn, size_t bytes) {
    if (bytes <= 48 * 1024) return ARV_OK;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e != cudaSuccess) return set_error(ARV_ERR_CUDA, "smem opt-in %zu B: %s", bytes, cudaGetErrorString(e));
    return ARV_OK;
}

}  // namespace arv

using namespace arv;

extern "C" {

int arv_constant_eval(const double *values, int64_t nvals, const double *u, double *out, int64_t n, void *stream) {
    if (nvals < 1) return set_error(ARV_ERR_CONFIG, "constant_eval: empty value table");
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    const int use_smem = nvals <= 8192;  // 64 KiB
    const size_t smem = use_smem ? sizeof(double) * nvals : 0;
    if (int rc = set_smem((const void *)k_constant_eval, smem)) return rc;
    k_constant_eval<<<eval_grid((const void *)k_constant_eval, n, smem), kEvalBlock, smem, as_stream(stream)>>>(values, nvals, use_smem, u, out, n);
    return finish("arv_constant_eval");
}

int arv_dyadic_index(const double *u, int64_t n, int64_t cap, int64_t *out, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_dyadic_index<<<eval_grid((const void *)k_dyadic_index, n, 0), kEvalBlock, 0, as_stream(stream)>>>(u, cap, reinterpret_cast<long long *>(out), n);
    return finish("arv_dyadic_index");
}

int arv_dyadic_index32(const float *u, int64_t n, int64_t cap, int64_t *out, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_dyadic_index32<<<eval_grid((const void *)k_dyadic_index32, n, 0), kEvalBlock, 0, as_stream(stream)>>>(u, cap, reinterpret_cast<long long *>(out), n);
    return finish("arv_dyadic_index32");
}

#define ARV_DEG_SWITCH(degree, MACRO) \
    switch (degree) {                 \
        MACRO(1) MACRO(2) MACRO(3) MACRO(4) MACRO(5)                    \
        default: return set_error(ARV_ERR_CONFIG, "polynomial degree must be in [1, 5], got %d", degree); \
    }

int arv_dyadic_eval(const double *coeffs, int degree, int64_t K1, const double *u, double *out, int64_t n,
                    void *stream) {
    if (K1 < 2 || K1 > 4096) return set_error(ARV_ERR_CONFIG, "dyadic_eval: bad interval count %lld", (long long)K1);
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    const size_t smem = sizeof(double) * (degree + 1) * K1;
    cudaStream_t s = as_stream(stream);
#define ARV_CASE(D)                                                                     \
    case D:                                                                             \
        if (int rc = set_smem((const void *)k_dyadic_eval<D>, smem)) return rc;          \
        k_dyadic_eval<D><<<eval_grid((const void *)k_dyadic_eval<D>, n, smem), kEvalBlock, smem, s>>>(coeffs, K1, u, out, n);          \
        break;
    ARV_DEG_SWITCH(degree, ARV_CASE)
#undef ARV_CASE
    return finish("arv_dyadic_eval");
}

int arv_dyadic_eval32(const float *coeffs, int degree, int64_t K1, const float *u, float *out, int64_t n,
                      void *stream) {
    if (K1 < 2 || K1 > 4096) return set_error(ARV_ERR_CONFIG, "dyadic_eval32: bad interval count %lld", (long long)K1);
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    const size_t smem = sizeof(float) * (degree + 1) * K1;
    cudaStream_t s = as_stream(stream);
#define ARV_CASE(D)                                                                     \
    case D:                                                                             \
        if (int rc = set_smem((const void *)k_dyadic_eval32<D>, smem)) return rc;        \
        k_dyadic_eval32<D><<<eval_grid((const void *)k_dyadic_eval32<D>, n, smem), kEvalBlock, smem, s>>>(coeffs, K1, u, out, n);        \
        break;
    ARV_DEG_SWITCH(degree, ARV_CASE)
#undef ARV_CASE
    return finish("arv_dyadic_eval32");
}

int arv_subdyadic_eval32(const float *coeffs, int degree, int K, int sub_bits, const float *u, float *out, int64_t n,
                         void *stream) {
    if (K < 1 || K > 40) return set_error(ARV_ERR_CONFIG, "octave count K must be in [1, 40], got %d", K);
    if (sub_bits < 0 || sub_bits > 5) return set_error(ARV_ERR_CONFIG, "sub_bits must be in [0, 5], got %d", sub_bits);
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    const size_t smem = sizeof(float) * (degree + 1) * ((size_t)(K + 1) << sub_bits);
    cudaStream_t s = as_stream(stream);
#define ARV_CASE(D)                                                                       \
    case D:                                                                               \
        k_subdyadic_eval32<D><<<eval_grid((const void *)k_subdyadic_eval32<D>, n, smem), kEvalBlock, smem, s>>>(coeffs, K, sub_bits, u, out, n); \
        break;
    ARV_DEG_SWITCH(degree, ARV_CASE)
#undef ARV_CASE
    return finish("arv_subdyadic_eval32");
}

int arv_ncchi2_eval(const double *stacks, int64_t n_knots, int degree, int64_t K1, double nu, const double *u,
                    const double *lam, int64_t nlam, double *out, int64_t n, void *stream) {
    if (n_knots < 2) return set_error(ARV_ERR_CONFIG, "need at least 2 knots, got %lld", (long long)n_knots);
    if (K1 < 2) return set_error(ARV_ERR_CONFIG, "ncchi2_eval: bad interval count");
    if (nlam != 1 && nlam != n) return set_error(ARV_ERR_CONFIG, "per-element lambda must match the shape of u");
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    const size_t bytes = sizeof(double) * 2 * n_knots * (degree + 1) * K1;
    const int use_smem = bytes <= 160 * 1024;
    const size_t smem = use_smem ? bytes : 0;
    cudaStream_t s = as_stream(stream);
#define ARV_CASE(D)                                                                                       \
    case D:                                                                                               \
        if (int rc = set_smem((const void *)k_ncchi2_eval<D>, smem)) return rc;                            \
        k_ncchi2_eval<D><<<eval_grid((const void *)k_ncchi2_eval<D>, n, smem), kEvalBlock, smem, s>>>(stacks, n_knots, K1, use_smem, nu, u, lam, nlam, out, n); \
        break;
    ARV_DEG_SWITCH(degree, ARV_CASE)
#undef ARV_CASE
    return finish("arv_ncchi2_eval");
}

int arv_gaussian_inv_cdf(const double *u, double *out, int64_t n, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_gauss_inv_cdf<<<eval_grid((const void *)k_gauss_inv_cdf, n, 0), kEvalBlock, 0, as_stream(stream)>>>(u, out, n);
    return finish("arv_gaussian_inv_cdf");
}

int arv_gaussian_inv_cdf32(const float *u, float *out, int64_t n, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_gauss_inv_cdf32<<<eval_grid((const void *)k_gauss_inv_cdf32, n, 0), kEvalBlock, 0, as_stream(stream)>>>(u, out, n);
    return finish("arv_gaussian_inv_cdf32");
}

}  // extern "C"

// Drop-in replacements of the reference kernel plugin (_kernels.pyx:16-143)
// on device arrays, plus the f32 octave x sub-interval evaluator and the
// AS241 exact quantile.  Element-wise, HBM-bound: tables are staged once per
// CTA in shared memory, inputs are read once and outputs written once.
#include "arv_common.cuh"
#include "arv_eval_dev.cuh"

namespace arv {

constexpr int kEvalBlock = 256;
constexpr int kEvalPerSM = 8;

static inline int eval_grid(int64_t n) { return stream_grid(n, kEvalBlock, kEvalPerSM); }

#define ARV_GRID_STRIDE(i, n)                                                               \
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)

// ------------------------------------------------------- constant_eval --
// _kernels.pyx:16-23: idx = (long long)(nvals * u), idx = min(idx, nvals-1).
__global__ void __launch_bounds__(kEvalBlock) k_constant_eval(const double *__restrict__ values, int64_t nvals,
                                                              int use_smem, const double *__restrict__ u,
                                                              double *__restrict__ out, int64_t n) {
    extern __shared__ double smd[];
    const double *tab = values;
    if (use_smem) {
        for (int i = threadIdx.x; i < nvals; i += blockDim.x) smd[i] = __ldg(values + i);
        __syncthreads();
        tab = smd;
    }
    const double scale = static_cast<double>(nvals);
    ARV_GRID_STRIDE(i, n) {
        long long idx = static_cast<long long>(__dmul_rn(scale, __ldcs(u + i)));
        idx = idx < nvals ? idx : nvals - 1;
        idx = idx < 0 ? 0 : idx;  // memory-safety clamp (u outside the (0,1) contract)
        __stcs(out + i, tab[idx]);
    }
}

// -------------------------------------------------------- dyadic_index --
__global__ void __launch_bounds__(kEvalBlock) k_dyadic_index(const double *__restrict__ u, int64_t cap,
                                                             long long *__restrict__ out, int64_t n) {
    ARV_GRID_STRIDE(i, n) __stcs(out + i, dyadic_idx64(__ldcs(u + i), cap));
}
__global__ void __launch_bounds__(kEvalBlock) k_dyadic_index32(const float *__restrict__ u, int64_t cap,
                                                               long long *__restrict__ out, int64_t n) {
    ARV_GRID_STRIDE(i, n) __stcs(out + i, dyadic_idx32(__ldcs(u + i), cap));
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
    ARV_GRID_STRIDE(i, n) {
        const double ui = __ldcs(u + i);
        const bool pred = ui < 0.5;
        const double v = pred ? ui : __dsub_rn(1.0, ui);
        long long idx = dyadic_idx64(v, cap);
        idx = idx < 0 ? 0 : idx;
        double z = smd[DEG * K1 + idx];
#pragma unroll
        for (int d = DEG - 1; d >= 0; --d) z = __dadd_rn(__dmul_rn(z, v), smd[d * K1 + idx]);
        __stcs(out + i, pred ? z : -z);
    }
}

template <int DEG>
__global__ void __launch_bounds__(kEvalBlock) k_dyadic_eval32(const float *__restrict__ coeffs, int64_t K1,
                                                              const float *__restrict__ u, float *__restrict__ out,
                                                              int64_t n) {
    extern __shared__ float smf[];
    for (int i = threadIdx.x; i < (DEG + 1) * K1; i += blockDim.x) smf[i] = __ldg(coeffs + i);
    __syncthreads();
    const long long cap = K1 - 1;
    ARV_GRID_STRIDE(i, n) {
        const float ui = __ldcs(u + i);
        const bool pred = ui < 0.5f;
        const float v = pred ? ui : __fsub_rn(1.0f, ui);
        long long idx = dyadic_idx32(v, cap);
        idx = idx < 0 ? 0 : idx;
        float z = smf[DEG * K1 + idx];
#pragma unroll
        for (int d = DEG - 1; d >= 0; --d) z = __fadd_rn(__fmul_rn(z, v), smf[d * K1 + idx]);
        __stcs(out + i, pred ? z : -z);
    }
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
    ARV_GRID_STRIDE(i, n) {
        const float ui = __ldcs(u + i);
        const bool pred = ui < 0.5f;
        const float v = pred ? ui : __fsub_rn(1.0f, ui);
        int e = static_cast<int>(__float_as_uint(v) >> shift) - base;
        e = min(max(e, 0), plane - 1);
        float z = smf[DEG * plane + e];
#pragma unroll
        for (int d = DEG - 1; d >= 0; --d) z = __fadd_rn(__fmul_rn(z, v), smf[d * plane + e]);
        __stcs(out + i, pred ? z : -z);
    }
}

// --------------------------------------------------------- ncchi2_eval --
// _kernels.pyx:96-143.  stacks (2, n_knots, DEG+1, K1): upper half at 0,
// lower at 1; knot bracketing j = min(floor(sqrt(nu/(lam+nu)) (n_knots-1)),
// n_knots-2), linear interpolation in t.  All IEEE (div/sqrt round-to-nearest).
template <int DEG>
__global__ void __launch_bounds__(kEvalBlock) k_ncchi2_eval(const double *__restrict__ stacks, int64_t n_knots,
                                                            int64_t K1, int use_smem, double nu,
                                                            const double *__restrict__ u,
                                                            const double *__restrict__ lam, int64_t nlam,
                                                            double *__restrict__ out, int64_t n) {
    extern __shared__ double smd[];
    const double *tab = stacks;
    if (use_smem) {
        const int64_t total = 2 * n_knots * (DEG + 1) * K1;
        for (int64_t i = threadIdx.x; i < total; i += blockDim.x) smd[i] = __ldg(stacks + i);
        __syncthreads();
        tab = smd;
    }
    ARV_GRID_STRIDE(i, n) {
        const double li = nlam == 1 ? __ldg(lam) : __ldcs(lam + i);
        __stcs(out + i, ncchi2_eval1<DEG>(tab, n_knots, K1, nu, __ldcs(u + i), li));
    }
}

// ---------------------------------------------------------- AS241 exact --
__global__ void __launch_bounds__(kEvalBlock) k_gauss_inv_cdf(const double *__restrict__ u, double *__restrict__ out,
                                                              int64_t n) {
    ARV_GRID_STRIDE(i, n) __stcs(out + i, as241_f64(__ldcs(u + i)));
}
__global__ void __launch_bounds__(kEvalBlock) k_gauss_inv_cdf32(const float *__restrict__ u, float *__restrict__ out,
                                                                int64_t n) {
    ARV_GRID_STRIDE(i, n) __stcs(out + i, as241_f32(__ldcs(u + i)));
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
    k_constant_eval<<<eval_grid(n), kEvalBlock, smem, as_stream(stream)>>>(values, nvals, use_smem, u, out, n);
    return finish("arv_constant_eval");
}

int arv_dyadic_index(const double *u, int64_t n, int64_t cap, int64_t *out, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_dyadic_index<<<eval_grid(n), kEvalBlock, 0, as_stream(stream)>>>(u, cap, reinterpret_cast<long long *>(out), n);
    return finish("arv_dyadic_index");
}

int arv_dyadic_index32(const float *u, int64_t n, int64_t cap, int64_t *out, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_dyadic_index32<<<eval_grid(n), kEvalBlock, 0, as_stream(stream)>>>(u, cap, reinterpret_cast<long long *>(out), n);
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
    const int grid = eval_grid(n);
    cudaStream_t s = as_stream(stream);
#define ARV_CASE(D)                                                                     \
    case D:                                                                             \
        if (int rc = set_smem((const void *)k_dyadic_eval<D>, smem)) return rc;          \
        k_dyadic_eval<D><<<grid, kEvalBlock, smem, s>>>(coeffs, K1, u, out, n);          \
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
    const int grid = eval_grid(n);
    cudaStream_t s = as_stream(stream);
#define ARV_CASE(D)                                                                     \
    case D:                                                                             \
        if (int rc = set_smem((const void *)k_dyadic_eval32<D>, smem)) return rc;        \
        k_dyadic_eval32<D><<<grid, kEvalBlock, smem, s>>>(coeffs, K1, u, out, n);        \
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
    const int grid = eval_grid(n);
    cudaStream_t s = as_stream(stream);
#define ARV_CASE(D)                                                                       \
    case D:                                                                               \
        k_subdyadic_eval32<D><<<grid, kEvalBlock, smem, s>>>(coeffs, K, sub_bits, u, out, n); \
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
    const int grid = eval_grid(n);
    cudaStream_t s = as_stream(stream);
#define ARV_CASE(D)                                                                                       \
    case D:                                                                                               \
        if (int rc = set_smem((const void *)k_ncchi2_eval<D>, smem)) return rc;                            \
        k_ncchi2_eval<D><<<grid, kEvalBlock, smem, s>>>(stacks, n_knots, K1, use_smem, nu, u, lam, nlam, out, n); \
        break;
    ARV_DEG_SWITCH(degree, ARV_CASE)
#undef ARV_CASE
    return finish("arv_ncchi2_eval");
}

int arv_gaussian_inv_cdf(const double *u, double *out, int64_t n, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_gauss_inv_cdf<<<eval_grid(n), kEvalBlock, 0, as_stream(stream)>>>(u, out, n);
    return finish("arv_gaussian_inv_cdf");
}

int arv_gaussian_inv_cdf32(const float *u, float *out, int64_t n, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_gauss_inv_cdf32<<<eval_grid(n), kEvalBlock, 0, as_stream(stream)>>>(u, out, n);
    return finish("arv_gaussian_inv_cdf32");
}

}  // extern "C"

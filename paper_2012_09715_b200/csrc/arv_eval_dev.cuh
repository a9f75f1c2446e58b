// Device evaluators shared by the drop-in kernels and the MLMC path kernels.
#pragma once

#include "arv_common.cuh"

namespace arv {

// _kernels.pyx:56-73 for one element; coefficient table `c` (DEG+1, K1).
// `pred` is the reference's u < 0.5 (callers with the PCG32 word pass it from
// an integer compare).
template <int DEG>
__device__ __forceinline__ double dyadic_eval1(const double *c, int64_t K1, double ui, bool pred) {
    const double v = pred ? ui : __dsub_rn(1.0, ui);
    long long idx = dyadic_idx64(v, K1 - 1);
    idx = idx < 0 ? 0 : idx;
    double z = c[DEG * K1 + idx];
#pragma unroll
    for (int d = DEG - 1; d >= 0; --d) z = __dadd_rn(__dmul_rn(z, v), c[d * K1 + idx]);
    return pred ? z : -z;
}
template <int DEG>
__device__ __forceinline__ double dyadic_eval1(const double *c, int64_t K1, double ui) {
    return dyadic_eval1<DEG>(c, K1, ui, ui < 0.5);
}

// Approximate-side Gaussian table of the path kernels: DEG >= 1 is a dyadic
// table (degree+1, K1) evaluated as dyadic_eval; DEG == 0 is a piecewise-
// constant table values[K1] evaluated as constant_eval (_kernels.pyx:16-23).
template <int DEG>
__device__ __forceinline__ double gauss_table_eval(const double *c, int64_t K1, double u, bool lower) {
    if constexpr (DEG == 0) {
        long long idx = static_cast<long long>(__dmul_rn(static_cast<double>(K1), u));
        idx = idx < K1 ? idx : K1 - 1;
        idx = idx < 0 ? 0 : idx;
        return c[idx];
    } else {
        return dyadic_eval1<DEG>(c, K1, u, lower);
    }
}
template <int DEG>
__device__ __forceinline__ double gauss_table_eval(const double *c, int64_t K1, double u) {
    return gauss_table_eval<DEG>(c, K1, u, u < 0.5);
}

// _kernels.pyx:96-143 for one element.  stacks (2, n_knots, DEG+1, K1):
// upper half at 0, lower at 1; knot bracketing j = min(floor(sqrt(nu /
// (lam + nu)) (n_knots - 1)), n_knots - 2); linear interpolation in t.
// All IEEE (div / sqrt round-to-nearest), separately rounded mul/add.
// The lambda-dependent half (shift, scale, knot bracket) is split out so a
// batch with one shared lambda computes it once per thread: the two IEEE
// square roots and the division dominate the per-element FP64 cost.
struct NcKnot {
    double shift, scale2, t;
    long long j;
};

__device__ __forceinline__ NcKnot ncchi2_knot(int64_t n_knots, double nu, double lam_i) {
    NcKnot k;
    k.shift = __dadd_rn(lam_i, nu);
    k.scale2 = __dmul_rn(2.0, __dsqrt_rn(k.shift));
    const double s = __dsqrt_rn(__ddiv_rn(nu, k.shift));
    const double g = __dmul_rn(s, static_cast<double>(n_knots - 1));
    long long j = static_cast<long long>(g);
    j = j < n_knots - 2 ? j : n_knots - 2;
    k.j = j < 0 ? 0 : j;
    k.t = __dsub_rn(g, static_cast<double>(k.j));
    return k;
}

template <int DEG>
__device__ __forceinline__ double ncchi2_eval_at(const double *tab, int64_t n_knots, int64_t K1, const NcKnot &k,
                                                 double ui) {
    const long long cap = K1 - 1;
    const long long sel = ui < 0.5 ? 1 : 0;
    const double v = sel ? ui : __dsub_rn(1.0, ui);
    long long idx = dyadic_idx64(v, cap);
    idx = idx < 0 ? 0 : idx;
    const int64_t knot = (DEG + 1) * K1;
    const double *t0 = tab + (sel * n_knots + k.j) * knot;
    const double *t1 = t0 + knot;
    double z0 = t0[DEG * K1 + idx];
    double z1 = t1[DEG * K1 + idx];
#pragma unroll
    for (int d = DEG - 1; d >= 0; --d) {
        z0 = __dadd_rn(__dmul_rn(z0, v), t0[d * K1 + idx]);
        z1 = __dadd_rn(__dmul_rn(z1, v), t1[d * K1 + idx]);
    }
    return __dadd_rn(k.shift, __dmul_rn(k.scale2, __dadd_rn(z0, __dmul_rn(k.t, __dsub_rn(z1, z0)))));
}

template <int DEG>
__device__ __forceinline__ double ncchi2_eval1(const double *tab, int64_t n_knots, int64_t K1, double nu, double ui,
                                               double lam_i) {
    return ncchi2_eval_at<DEG>(tab, n_knots, K1, ncchi2_knot(n_knots, nu, lam_i), ui);
}

// Warm starts only (not the reference's arithmetic): the knot bracket and the
// scale 2 sqrt(lam + nu) from f32 reciprocal square roots -- relative error
// ~1e-7, far below the table's own ~1e-3 -- instead of two IEEE f64 square
// roots and a division.
__device__ __forceinline__ NcKnot ncchi2_knot_warm(int64_t n_knots, double nu, double lam_i) {
    NcKnot k;
    k.shift = lam_i + nu;
    const float sf = static_cast<float>(k.shift);
    const float r = rsqrtf(sf);
    k.scale2 = static_cast<double>(2.0f * sf * r);
    const float g = sqrtf(static_cast<float>(nu)) * r * static_cast<float>(n_knots - 1);
    long long j = static_cast<long long>(g);
    j = j < n_knots - 2 ? j : n_knots - 2;
    k.j = j < 0 ? 0 : j;
    k.t = static_cast<double>(g - static_cast<float>(k.j));
    return k;
}
template <int DEG>
__device__ __forceinline__ double ncchi2_warm1(const double *tab, int64_t n_knots, int64_t K1, double nu, double ui,
                                               double lam_i) {
    return ncchi2_eval_at<DEG>(tab, n_knots, K1, ncchi2_knot_warm(n_knots, nu, lam_i), ui);
}

}  // namespace arv

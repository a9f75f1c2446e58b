// Device non-central chi-squared CDF / density / quantile (f64).
//
// Replaces, for the CIR exact transition, the reference's
// ncchi2_inv_cdf_batch per-element-lambda path (exact_dist.py:381-461):
// bisection-safeguarded Newton (_vector_newton, exact_dist.py:348-378) in the
// bracket [0, lam + nu + 20 sqrt(2(lam+nu)) + 100] with the tolerance
// tol_f = min(1e-9, max(1e-13, 1e-4 min(u, 1-u))) and the residual contract
// |F(x) - u| <= 1e-8 (exact_dist.py:452-460).  The reference evaluates F with
// scipy's CDFLIB chndtr; here F is the Poisson mixture of regularized lower
// incomplete gammas (the series of exact_dist.py:215-235),
//     F(x; nu, lam) = sum_j Pois(j; h) P(a0 + j, y),   h = lam/2, a0 = nu/2, y = x/2,
// and the density f(x) = 1/2 sum_j Pois(j; h) G(a0 + j - 1, y) with
// G(a, y) = y^a e^-y / Gamma(a + 1).
//
// Evaluation is ONE downward sweep over the index j with no incomplete-gamma
// series or continued fraction: P(a, y) = sum_{n >= 0} G(a + n, y), so
// starting at an index J where G(a0 + J, y) is negligible (above both the
// Poisson window and y + 9 sqrt(y)) and adding
//     G(a0 + j - 1) = G(a0 + j) (a0 + j) / y
// on the way down yields every P(a0 + j, y) as a sum of positive terms.  The
// Poisson weights join at the window top k + 9 sqrt(h) + 10 (neglected mass
// < 1e-17) through p_{j-1} = p_j j / h and are renormalised by their sum.
// Per term ~9 FP64 operations, no division, no table load, no transcendental,
// and every lane runs the same loop body (the earlier mode-centred version
// with series / continued fraction for the mode term diverged 3:1 across
// lanes: 172 ms -> 64 ms for the CIR level-6 kernel).  The only per-CDF
// transcendentals are two exp and two log, with lgamma(j + 1) and
// lgamma(a0 + j + 1) from per-CTA shared tables (j < kNcTab).
//
// Accuracy: P carries the relative rounding of exp/lgamma at J (~1e-12 at
// lambda ~ 250), an absolute error well inside the 1e-8 residual contract;
// Newton converges on this F itself, so tol_f is met on the device CDF.
#pragma once

#include "arv_common.cuh"

namespace arv {

constexpr int kNcTab = 1024;

struct NcTables {
    const double *lg_j;   // lgamma(j + 1)
    const double *lg_aj;  // lgamma(a0 + j + 1)
    double a0;

    __device__ __forceinline__ double lgj(int j) const {
        return j < kNcTab ? lg_j[j] : lgamma(static_cast<double>(j) + 1.0);
    }
    __device__ __forceinline__ double lgaj(int j) const {
        return j < kNcTab ? lg_aj[j] : lgamma(a0 + static_cast<double>(j) + 1.0);
    }
};

// Fill the tables in shared memory (kNcSmemDoubles doubles) for a0 = nu / 2.
constexpr int kNcSmemDoubles = 2 * kNcTab;
__device__ inline NcTables nc_tables_init(double *sm, double nu) {
    const double a0 = 0.5 * nu;
    for (int j = threadIdx.x; j < kNcTab; j += blockDim.x) {
        sm[j] = lgamma(static_cast<double>(j) + 1.0);
        sm[kNcTab + j] = lgamma(a0 + static_cast<double>(j) + 1.0);
    }
    __syncthreads();
    return {sm, sm + kNcTab, a0};
}

struct NcCdf {
    double resid;  // F(x) - u
    double pdf;
};

// F(x) - u and f(x) for x > 0.
__device__ inline NcCdf ncchi2_cdf_minus(const NcTables &t, double x, double lam, double u) {
    const double y = 0.5 * x;
    const double a0 = t.a0;
    const double h = 0.5 * lam;
    const double kd = floor(h);
    const int k = static_cast<int>(kd);
    const int wp = h < 1e-2 ? 8 : static_cast<int>(9.0 * sqrt(h)) + 10;
    const int top = k + wp;
    const int bot = k - wp > 0 ? k - wp : 0;
    const int jy = static_cast<int>(ceil(y - a0)) + static_cast<int>(9.0 * sqrt(y)) + 10;
    const int J = jy > top ? jy : top;
    const double inv_y = 1.0 / y;
    const double inv_h = h > 0.0 ? 1.0 / h : 0.0;
    double G = exp((a0 + static_cast<double>(J)) * log(y) - y - t.lgaj(J));  // G(a0 + J)
    double P = G;                                                           // P(a0 + J) ~ G(a0 + J)
    double jd = static_cast<double>(J);
    for (int j = J; j > top; --j) {  // above the Poisson window: P and G only
        G *= (a0 + jd) * inv_y;
        P += G;
        jd -= 1.0;
    }
    // Poisson weight at the window top (h > 0); h == 0 is the central law (p_0 = 1)
    double p = h > 0.0 ? exp(-h + jd * log(h) - t.lgj(top)) : (top == 0 ? 1.0 : 0.0);
    double wsum = 0.0, acc = 0.0, dens = 0.0;
    for (int j = top; j >= bot; --j) {
        wsum += p;
        acc += p * P;
        const double Gm = G * (a0 + jd) * inv_y;  // G(a0 + j - 1)
        dens += p * Gm;
        P += Gm;
        G = Gm;
        p = h > 0.0 ? p * jd * inv_h : (j == 1 ? 1.0 : 0.0);
        jd -= 1.0;
    }
    return {acc / wsum - u, 0.5 * dens / wsum};
}

struct NcQuantile {
    double x;
    double resid;  // |F(x) - u|
};

// exact_dist.py:381-461 contract, per element, warm start x0 (<= 0: mean).
__device__ inline NcQuantile ncchi2_quantile(const NcTables &t, double u, double nu, double lam, double x0) {
    const double one_minus_u = 1.0 - u;
    double hi = lam + nu + 20.0 * sqrt(2.0 * (lam + nu)) + 100.0;
    double lo = 0.0;
    const double tol_f = fmin(1e-9, fmax(1e-13, 1e-4 * fmin(u, one_minus_u)));
    double x = x0 > 0.0 ? x0 : lam + nu;
    x = fmin(fmax(x, 1e-8), hi);
    NcCdf c = ncchi2_cdf_minus(t, x, lam, u);
    for (int it = 0; it < 80; ++it) {
        if (fabs(c.resid) <= tol_f) break;
        if (c.resid > 0.0) hi = x;
        else lo = x;
        double xn = x - c.resid / c.pdf;
        if (!isfinite(xn) || xn <= lo || xn >= hi) xn = 0.5 * (lo + hi);
        x = xn;
        c = ncchi2_cdf_minus(t, x, lam, u);
        if (hi - lo < 1e-15 * hi) break;
    }
    return {x, fabs(c.resid)};
}

}  // namespace arv

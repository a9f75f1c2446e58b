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
//     F(x; nu, lam) = sum_j Pois(j; lam/2) P(nu/2 + j, x/2),
// evaluated from the Poisson mode outwards with the two-term recurrences
//     P(a+1, y) = P(a, y) - G(a),  G(a) = y^a e^-y / Gamma(a+1),
//     G(a+1) = G(a) y / (a+1),     Pois(j+1) = Pois(j) h / (j+1),
// (the Benton-Krishnamoorthy organisation of Ding's series), so one pass
// yields F and the density f(x) = 1/2 sum_j Pois(j) G(nu/2 + j - 1).  The
// mode term P(a, y) comes from the power series (y < a+1) or the Lentz
// continued fraction of Q (y >= a+1); whichever side is smaller is carried
// through the recurrence, so tails keep their relative accuracy.  Poisson
// weights are renormalised by their computed sum, cancelling the common
// rounding of exp/lgamma in the mode weight.
//
// Speed: every per-term division of the recurrences uses a per-CTA shared
// table -- 1/j, 1/(nu/2 + j), lgamma(j + 1), lgamma(nu/2 + j + 1) for
// j < kNcTab -- so the inner loops are multiply/add only; indices past the
// table fall back to direct division / lgamma.
#pragma once

#include "arv_common.cuh"

namespace arv {

constexpr int kNcTab = 1024;

struct NcTables {
    const double *inv_j;   // 1 / j            (inv_j[0] unused)
    const double *inv_aj;  // 1 / (a0 + j)
    const double *lg_j;    // lgamma(j + 1)
    const double *lg_aj;   // lgamma(a0 + j + 1)
    double a0;

    __device__ __forceinline__ double rj(long long j) const { return j < kNcTab ? inv_j[j] : 1.0 / j; }
    __device__ __forceinline__ double raj(long long j) const {
        return j < kNcTab ? inv_aj[j] : 1.0 / (a0 + static_cast<double>(j));
    }
    __device__ __forceinline__ double lgj(long long j) const {
        return j < kNcTab ? lg_j[j] : lgamma(static_cast<double>(j) + 1.0);
    }
    __device__ __forceinline__ double lgaj(long long j) const {
        return j < kNcTab ? lg_aj[j] : lgamma(a0 + static_cast<double>(j) + 1.0);
    }
};

// Fill the tables in shared memory (4 * kNcTab doubles) for a0 = nu / 2.
__device__ inline NcTables nc_tables_init(double *sm, double nu) {
    const double a0 = 0.5 * nu;
    for (int j = threadIdx.x; j < kNcTab; j += blockDim.x) {
        sm[j] = j ? 1.0 / j : 0.0;
        sm[kNcTab + j] = 1.0 / (a0 + j);
        sm[2 * kNcTab + j] = lgamma(static_cast<double>(j) + 1.0);
        sm[3 * kNcTab + j] = lgamma(a0 + static_cast<double>(j) + 1.0);
    }
    __syncthreads();
    return {sm, sm + kNcTab, sm + 2 * kNcTab, sm + 3 * kNcTab, a0};
}

#ifndef ARV_NC_SERIES_ONLY
#define ARV_NC_SERIES_ONLY 1
#endif

struct GammaPQ {
    double small;  // P if lower, else Q
    bool lower;
    double G;      // y^a e^-y / Gamma(a+1)
};

// Regularized incomplete gamma at (a, y) = (a0 + k, y), y > 0.
__device__ inline GammaPQ gamma_pq(const NcTables &t, long long k, double y, double log_y) {
    const double a = t.a0 + static_cast<double>(k);
    const double G = exp(a * log_y - y - t.lgaj(k));
    GammaPQ r;
    r.G = G;
    // Series for every lane (also y >= a + 1, where its terms first grow):
    // one code path per warp instead of series/continued-fraction divergence,
    // and the P side carries an absolute error ~1e-16 x terms, well inside the
    // quantile tolerance tol_f >= 1e-13 (which is absolute, exact_dist.py:409).
    if (ARV_NC_SERIES_ONLY || y < a + 1.0) {
        // P = G * sum_{n>=0} y^n / ((a+1)...(a+n)),  1/(a+n) = 1/(a0+k+n)
        double sum = 1.0, term = 1.0;
        int n = static_cast<int>(k) + 1;
        bool done = false;
        for (; n < kNcTab; ++n) {  // 1/(a0 + n) from the table
            term *= y * t.inv_aj[n];
            sum += term;
            if (term < sum * 1e-17) {
                done = true;
                break;
            }
        }
        if (!done) {
            double an = t.a0 + static_cast<double>(n);
            for (int guard = 0; guard < 4000; ++guard, an += 1.0) {
                term *= y / an;
                sum += term;
                if (term < sum * 1e-17) break;
            }
        }
        r.small = G * sum;
        r.lower = true;
    } else {
        // Q = (G a / y) * y / (y + 1 - a - 1(1-a)/(y + 3 - a - ...)) (modified Lentz)
        const double tiny = 1e-300;
        double b = y + 1.0 - a;
        double c = 1.0 / tiny;
        double d = 1.0 / b;
        double h = d;
        for (int i = 1; i < 2000; ++i) {
            const double an = -i * (i - a);
            b += 2.0;
            d = an * d + b;
            if (fabs(d) < tiny) d = tiny;
            c = b + an / c;
            if (fabs(c) < tiny) c = tiny;
            d = 1.0 / d;
            const double del = d * c;
            h *= del;
            if (fabs(del - 1.0) < 1e-16) break;
        }
        r.small = G * a * h;  // e^-y y^a / Gamma(a) * h
        r.lower = false;
    }
    return r;
}

struct NcCdf {
    double resid;  // F(x) - u, computed on the accurate side
    double pdf;
};

// Poisson window forward from the mode, j = k+1, k+2, ...: the carried side
// S_j (P_j if LOWER, Q_j otherwise) changes by G_{j-1} = G(a0 + j - 1), which
// is also the density term.  The table phase (j < kNcTab) is multiply/add
// only; a second loop with divisions covers windows past the tables.  Loop
// counters stay 32-bit and j is tracked as a double (no I2F per term).
template <bool LOWER>
__device__ __forceinline__ void nc_forward(const NcTables &t, long long k, double kd, double h, double y, double pk,
                                           double S, double G, double &wsum, double &acc, double &dens) {
    double p = pk, jd = kd;
    int j = static_cast<int>(k) + 1;
    for (; j < kNcTab; ++j) {
        jd += 1.0;
        p *= h * t.inv_j[j];
        S = LOWER ? fmax(S - G, 0.0) : S + G;
        dens += p * G;
        G *= y * t.inv_aj[j];
        wsum += p;
        acc += p * S;
        if (p < 1e-18 && jd > h) return;
    }
    for (int guard = 0; guard < 200000; ++guard) {
        jd += 1.0;
        p *= h / jd;
        S = LOWER ? fmax(S - G, 0.0) : S + G;
        dens += p * G;
        G *= y / (t.a0 + jd);
        wsum += p;
        acc += p * S;
        if (p < 1e-18 && jd > h) return;
    }
}

// Backward from the mode, j = k-1, ..., 0: G_j = G_{j+1} (a0 + j + 1) / y,
// the carried side changes by G_j, the density term is G_{j-1}.
template <bool LOWER>
__device__ __forceinline__ void nc_backward(double a0, long long k, double kd, double inv_h, double inv_y, double pk,
                                            double S, double G, double &wsum, double &acc, double &dens) {
    double p = pk, jd = kd;  // jd = j + 1 at the top of each iteration
    for (long long j = k - 1; j >= 0; --j) {
        p *= jd * inv_h;
        const double aj = a0 + jd;  // a0 + j + 1
        G *= aj * inv_y;
        S = LOWER ? S + G : fmax(S - G, 0.0);
        wsum += p;
        acc += p * S;
        dens += p * G * (aj - 1.0) * inv_y;
        jd -= 1.0;
        if (p < 1e-18) return;
    }
}

// F(x) - u and f(x) for x > 0.  `one_minus_u` is exact for u >= 1/2.
__device__ inline NcCdf ncchi2_cdf_minus(const NcTables &t, double x, double lam, double u, double one_minus_u) {
    const double y = 0.5 * x;
    const double a0 = t.a0;
    const double h = 0.5 * lam;
    const double kd = floor(h);
    const long long k = static_cast<long long>(kd);
    const double pk = h > 0.0 ? exp(-h + kd * log(h) - t.lgj(k)) : 1.0;
    const double inv_y = 1.0 / y;
    const double inv_h = h > 0.0 ? 1.0 / h : 0.0;

    const GammaPQ g = gamma_pq(t, k, y, log(y));
    const bool lower = g.lower;
    // Mode term.  Carried side S_j: P_j (lower) or Q_j (upper).
    double wsum = pk;
    double acc = pk * g.small;
    // density: 1/2 pk G(a0 + k - 1) = 1/2 pk G_k (a0 + k) / y
    double dens = pk * g.G * (a0 + kd) * inv_y;

    if (lower) {
        nc_forward<true>(t, k, kd, h, y, pk, g.small, g.G, wsum, acc, dens);
        nc_backward<true>(a0, k, kd, inv_h, inv_y, pk, g.small, g.G, wsum, acc, dens);
    } else {
        nc_forward<false>(t, k, kd, h, y, pk, g.small, g.G, wsum, acc, dens);
        nc_backward<false>(a0, k, kd, inv_h, inv_y, pk, g.small, g.G, wsum, acc, dens);
    }
    NcCdf r;
    const double side = acc / wsum;
    r.resid = lower ? side - u : one_minus_u - side;
    r.pdf = 0.5 * dens / wsum;
    return r;
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
    NcCdf c = ncchi2_cdf_minus(t, x, lam, u, one_minus_u);
    for (int it = 0; it < 80; ++it) {
        if (fabs(c.resid) <= tol_f) break;
        if (c.resid > 0.0) hi = x;
        else lo = x;
        double xn = x - c.resid / c.pdf;
        if (!isfinite(xn) || xn <= lo || xn >= hi) xn = 0.5 * (lo + hi);
        x = xn;
        c = ncchi2_cdf_minus(t, x, lam, u, one_minus_u);
        if (hi - lo < 1e-15 * hi) break;
    }
    return {x, fabs(c.resid)};
}

}  // namespace arv

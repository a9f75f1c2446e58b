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
// Poisson window and y + 8 sqrt(y)) and adding
//     G(a0 + j - 1) = G(a0 + j) (a0 + j) / y
// on the way down yields every P(a0 + j, y) as a sum of positive terms.  The
// Poisson weights join at the window top k + 8 sqrt(h) + 10 (neglected mass
// < ~1e-15) through p_{j-1} = p_j j / h and are renormalised by their sum.
// Per window term 9 FP64 operations (the factor (a0 + j)/y is one FMA of the
// exact index), no division, no table load, no transcendental, and every
// lane runs the same loop body.  Everything that depends on lambda alone
// (window, Poisson weight at its top) is set up once per quantile solve.
//
// The two starting values G(a0 + J, y) and Pois(top; h) are densities of the
// form lam^x e^-lam / Gamma(x + 1) evaluated far from the mode.  Computed as
// exp(x log lam - lam - lgamma(x + 1)) their relative error is the exponent's
// magnitude times epsilon (5e-12 at lam ~ 1e4), so they use the saddle-point
// form of C. Loader ("Fast and accurate computation of binomial
// probabilities", 2000): exp(-stirlerr(x) - bd0(x, lam)) / sqrt(2 pi x) with
// the Stirling remainder stirlerr and the deviance bd0 = x log(x/lam) + lam - x
// summed by its series near x = lam -- relative error a few epsilon at any
// magnitude, and no per-CTA lgamma tables.
#pragma once

#include "arv_common.cuh"

#include "arv_logtab.cuh"

#ifndef ARV_NC_FAST_LOG
#define ARV_NC_FAST_LOG 1
#endif

namespace arv {

// stirlerr(n) = log Gamma(n + 1) - (n + 1/2) log n + n - log sqrt(2 pi):
// exact values at n = 0..15 (50-digit evaluation), the asymptotic series
// 1/(12n) - 1/(360n^3) + ... (5 terms, |error| < 2e-14 for n > 10) above,
// lgamma for the remaining non-integer n <= 10 (not reached by the sweep:
// its arguments are a0 + J > 10 and the integer window top).
static __constant__ double kStirlerrInt[16] = {
    0.0, 8.1061466795327258e-2, 4.1340695955409294e-2, 2.7677925684998339e-2,
    2.0790672103765093e-2, 1.6644691189821192e-2, 1.3876128823070748e-2, 1.1896709945891770e-2,
    1.0411265261972096e-2, 9.2554621827127329e-3, 8.3305634333628713e-3, 7.5736754879518408e-3,
    6.9428401072095299e-3, 6.4089941880042071e-3, 5.9513701127588477e-3, 5.5547335519628014e-3};

// log(x) for a positive normal x from the level kernels' 128-bucket table
// (arv_logtab.cuh; the same evaluation as g2::neg_log in arv_mlmc.cu): 9 FP64
// operations where CUDA's log() takes ~25 plus ~30 other instructions.
// Absolute error ~2^-58 + 1.1 ulp of the result; its uses here are
// log(2 pi x) with x >= 1 and log(x / m) with |log| >= 0.2.
__device__ __forceinline__ double nc_log(double v) {
#if ARV_NC_FAST_LOG
    const int hi = __double2hiint(v);
    if (static_cast<unsigned>(hi - 0x00100000) >= 0x7FE00000u) return log(v);  // zero, subnormal, negative, inf, nan
    const int ne = 1023 - (hi >> 20);
    const double2 tj = __ldg(kLogTab + ((hi >> 13) & 127));
    const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(v));
    const double r = fma(m, tj.x, -1.0);
    double q = fma(r, -1.0 / 6.0, 0.2);
    q = fma(q, r, -0.25);
    q = fma(q, r, 1.0 / 3.0);
    q = fma(q, r, -0.5);
    const double lp = fma(r * r, q, r);
    return lp - fma(static_cast<double>(ne), 0.6931471805599453094, tj.y);
#else
    return log(v);
#endif
}

__device__ inline double nc_stirlerr(double n) {
    if (n <= 15.0 && n == floor(n)) return kStirlerrInt[static_cast<int>(n)];
    if (n > 10.0) {
        const double r = 1.0 / n, r2 = r * r;
        return r * (1.0 / 12.0 - r2 * (1.0 / 360.0 - r2 * (1.0 / 1260.0 - r2 * (1.0 / 1680.0 - r2 * (1.0 / 1188.0)))));
    }
    constexpr double kLnSqrt2Pi = 0.918938533204672741780329736406;
    return lgamma(n + 1.0) - (n + 0.5) * log(n) + n - kLnSqrt2Pi;
}

// bd0(x, m) = x log(x / m) + m - x; near x = m by its series in
// v = (x - m)/(x + m): (x - m) v + 2 x v (v^2/3 + v^4/5 + ...), |v| < 0.1,
// 8 terms (v^16/17 < 1e-17 of the leading term)
__device__ inline double nc_bd0(double x, double m) {
    const double d = x - m;
    if (fabs(d) < 0.1 * (x + m)) {
        const double v = d / (x + m);
        const double v2 = v * v;
        double t = 1.0 / 17.0;
        t = fma(t, v2, 1.0 / 15.0);
        t = fma(t, v2, 1.0 / 13.0);
        t = fma(t, v2, 1.0 / 11.0);
        t = fma(t, v2, 1.0 / 9.0);
        t = fma(t, v2, 1.0 / 7.0);
        t = fma(t, v2, 1.0 / 5.0);
        t = fma(t, v2, 1.0 / 3.0);
        return fma(2.0 * x * v, v2 * t, d * v);
    }
    return x * nc_log(x / m) + m - x;
}

// log(m^x e^-m / Gamma(x + 1)) for real x >= 0, m >= 0
__device__ inline double nc_logdens(double x, double m) {
    if (m <= 0.0) return x == 0.0 ? 0.0 : -INFINITY;
    if (x == 0.0) return -m;
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    return -nc_stirlerr(x) - nc_bd0(x, m) - 0.5 * nc_log(kTwoPi * x);
}

struct NcCdf {
    double resid;  // F(x) - u
    double pdf;    // f(x) = S_1 / 2
    double s0;     // S_0 = sum_j Pois(j; h) G(a0 + j, y): the density of nu + 2, times 2
};

// Half-width of the Poisson window and height of the gamma sweep above y, in
// standard deviations (+10 terms).  8 sigma (the CDF entry points and tail
// quantiles): within 2.1e-13 of CDFLIB everywhere tested.  7 sigma (quantiles
// with min(u, 1-u) >= 1e-6, i.e. tol_f >= 1e-10): within ~1.1e-12 -- two
// orders below those tolerances and inside the reference's own 5e-12
// series-vs-CDFLIB bound (test_exact_dist.py:154-160) -- and 12% fewer terms.
#ifndef ARV_NC_SIGMAS
#define ARV_NC_SIGMAS 8.0
#endif
#ifndef ARV_NC_SIGMAS_BULK
#define ARV_NC_SIGMAS_BULK 7.0
#endif
#ifndef ARV_NC_NARROW_START
#define ARV_NC_NARROW_START 1
#endif
#ifndef ARV_NC_SIGMAS_START
#define ARV_NC_SIGMAS_START 6.0
#endif
constexpr double kNcSigmas = ARV_NC_SIGMAS;
constexpr double kNcSigmasBulk = ARV_NC_SIGMAS_BULK;
// First sweep of a bulk solve: it only places the Taylor step, whose result
// the full-width verification sweep then checks against tol_f >= 1e-10, so a
// 6-sigma window (truncation ~1e-11..1e-10) suffices there.
constexpr double kNcSigmasStart = ARV_NC_SIGMAS_START;

#ifndef ARV_NC_BLOCK
#define ARV_NC_BLOCK 128  // terms per block of incremental factors (0: exact factors every term)
#endif
#ifndef ARV_NC_BLOCK_MAXW
#define ARV_NC_BLOCK_MAXW 512  // longest window that uses the blocks
#endif

// The lambda-only part of the CDF: Poisson window [bot, top] around
// k = floor(lambda/2) and the weight at its top.  Fixed during a quantile
// solve, so it is computed once per (u, lambda), not once per Newton step.
struct NcLam {
    double h, inv_h, p_top, sigmas;
    int top, bot;
    bool blocked;  // bulk quantile solve: incremental sweep factors allowed
    int top_n, bot_n;  // narrower window for a bulk solve's first (Taylor-start) sweep
};

__device__ inline NcLam nc_lam(double lam, double sigmas = kNcSigmas) {
    NcLam L;
    L.h = 0.5 * lam;
    L.sigmas = sigmas;
    const int k = static_cast<int>(floor(L.h));
    // window extents are integer heuristics: f32 square roots suffice
    const int wp = L.h < 1e-2 ? 8 : static_cast<int>(static_cast<float>(sigmas) * sqrtf(static_cast<float>(L.h))) + 10;
    L.top = k + wp;
    L.bot = k - wp > 0 ? k - wp : 0;
    L.inv_h = L.h > 0.0 ? 1.0 / L.h : 0.0;
    L.p_top = L.h > 0.0 ? exp(nc_logdens(static_cast<double>(L.top), L.h)) : 0.0;
    L.blocked = sigmas < kNcSigmas && (L.top - L.bot + 1) <= ARV_NC_BLOCK_MAXW;
    const int wn = L.h < 1e-2 ? 8 : static_cast<int>(static_cast<float>(kNcSigmasStart) * sqrtf(static_cast<float>(L.h))) + 10;
    L.top_n = k + wn < L.top ? k + wn : L.top;
    L.bot_n = k - wn > L.bot ? k - wn : L.bot;
    return L;
}

// F(x) - u for x > 0, a0 = nu / 2.  FULL: also the density f(x) = S_1 / 2
// and S_0 (for the Taylor step).  !FULL (a verification evaluation of the
// same solve): F only -- 7 instead of 9 FP64 operations per window term.
// The Poisson weights are not renormalised by their window sum: p_top is
// Loader's saddle-point pmf (a few ulp), the
// window drops < 1e-15 of the Poisson mass, and the downward recurrence
// drifts by ~(window length) ulp, so F moves by < 1e-13 and one FP64
// operation per term is saved.
template <bool FULL>
__device__ inline NcCdf ncchi2_cdf_sweep(double a0, double x, const NcLam &L, double u, double &inv_w,
                                         const bool NARROW = false) {
    const double y = 0.5 * x;
    const int top = NARROW ? L.top_n : L.top, bot = NARROW ? L.bot_n : L.bot;
    const float sig = NARROW ? static_cast<float>(kNcSigmasStart) : static_cast<float>(L.sigmas);
    const int jy = static_cast<int>(ceil(y - a0)) + static_cast<int>(sig * sqrtf(static_cast<float>(y))) + 10;
    int j = jy > top ? jy : top;
    const double inv_y = 1.0 / y;
    const double a0y = a0 * inv_y;
    double jd = static_cast<double>(j);
    // G(a0 + J).  Far left tail (y << a0 + J) it underflows and the recurrence
    // would stay at zero: walk down in log space to the first representable
    // term; everything above it is below e^-700 of the retained terms.
    double lg = nc_logdens(a0 + jd, y);
    while (lg < -700.0 && j > 0) {
        lg += log(fma(jd, inv_y, a0y));
        jd -= 1.0;
        --j;
    }
    double G = exp(lg);
    double P = G;                    // P(a0 + j) ~ G(a0 + j)
#if ARV_NC_BLOCK
    if (L.blocked && j - top <= ARV_NC_BLOCK) {  // bulk: incremental factor (see the window loop)
        double f = fma(jd, inv_y, a0y);
        jd -= static_cast<double>(j > top ? j - top : 0);
        for (; j > top; --j) {
            G *= f;
            P += G;
            f -= inv_y;
        }
    }
#endif
    for (; j > top; --j) {           // above the Poisson window: P and G only
        G *= fma(jd, inv_y, a0y);    // G(a0 + j - 1) = G(a0 + j) (a0 + j) / y
        P += G;
        jd -= 1.0;
    }
    if (L.h > 0.0) {
        const double inv_h = L.inv_h;
        double p = L.p_top;
        if (NARROW) {  // Poisson weight at the narrow window top
            for (int i = L.top; i > top; --i) p *= static_cast<double>(i) * inv_h;
        }
        double acc = 0.0, dens = 0.0, s0 = 0.0;
        for (int i = top; i > j && i >= bot; --i) {  // window indices whose gamma terms underflowed
            p *= static_cast<double>(i) * inv_h;
        }
        auto term = [&](double fj, double rj) {
            acc = fma(p, P, acc);
            const double Gm = G * fj;  // G(a0 + j - 1)
            if constexpr (FULL) {
                s0 = fma(p, G, s0);
                dens = fma(p, Gm, dens);
            }
            P += Gm;
            G = Gm;
            p *= rj;
        };
#if ARV_NC_BLOCK
        // The two per-term factors (a0 + j)/y and j/h step down by 1/y and 1/h.
        // Within blocks of ARV_NC_BLOCK terms they are updated
        // by subtraction -- one FP64 operation per term fewer than recomputing
        // both from the exact index -- and re-derived from the index at each
        // block start.  A factor then carries at most ARV_NC_BLOCK roundings and
        // the product of W factors drifts by at most ~W * ARV_NC_BLOCK / 2
        // roundings.  Used only for bulk quantile solves (7-sigma windows,
        // tol_f >= 1e-10) with windows up to ARV_NC_BLOCK_MAXW terms (lambda up
        // to ~2500): their CDF error grows from <= 2.2e-13 to <= 7.9e-13 against
        // CDFLIB (nu in {1, 2, 7.3}, lambda <= 1000), far below their
        // tolerance.  Tail solves and the CDF entry point keep exact factors.
        if (L.blocked) {
            while (j >= bot) {
                double f = fma(jd, inv_y, a0y), r = jd * inv_h;
                const int nb = j - bot + 1 < ARV_NC_BLOCK ? j - bot + 1 : ARV_NC_BLOCK;
                for (int t = 0; t < nb; ++t) {
                    term(f, r);
                    f -= inv_y;
                    r -= inv_h;
                }
                j -= nb;
                jd -= static_cast<double>(nb);
            }
        }
#endif
        for (; j >= bot; --j) {
            term(fma(jd, inv_y, a0y), jd * inv_h);
            jd -= 1.0;
        }
        if constexpr (FULL) inv_w = 1.0;
        return {fma(acc, inv_w, -u), 0.5 * dens * inv_w, s0 * inv_w};
    }
    // h == 0: the central law, F = P(a0, y), f = G(a0 - 1, y) / 2
    for (; j > 0; --j) {
        G *= fma(jd, inv_y, a0y);
        P += G;
        jd -= 1.0;
    }
    return {P - u, 0.5 * G * a0y, G};
}

__device__ inline NcCdf ncchi2_cdf_minus(double a0, double x, const NcLam &L, double u) {
    double inv_w;
    return ncchi2_cdf_sweep<true>(a0, x, L, u, inv_w);
}

struct NcQuantile {
    double x;
    double resid;  // |F(x) - u|
};

// Degree of the Taylor-polynomial step (0: Newton / Halley steps instead).
#ifndef ARV_NC_TAYLOR
#define ARV_NC_TAYLOR 4
#endif

// One high-order step from a CDF evaluation.  With y = x/2 and
// S_k = sum_j Pois(j; h) G(a0 + j - k, y) (S_k is twice the density of
// nu - 2k + 2 degrees of freedom), d/dy F = S_1 and d/dy S_k = S_{k+1} - S_k,
// so the n-th y-derivative of F is the forward difference Delta^{n-1} S_1.
// The S_k obey the Bessel recurrence in the order
//     S_{k+1} = (h S_{k-1} + (a0 - k) S_k) / y        (I_{m-1} - I_{m+1} = 2m/z I_m,
// stable in this direction), so the sweep's S_0 and S_1 give every Taylor
// coefficient of F around x for a few FP64 operations.  The step is the root
// of the degree-DEG Taylor polynomial nearest 0 (Newton on the polynomial from
// the plain Newton step, registers only).  From the table warm start its
// error is ~(warm-start error)^(DEG+1): for config 5 (DEG = 4), 99.99% of
// solves meet tol_f after this one step, so a solve costs 2 CDF evaluations
// (start + verification) instead of the 2.98 of Newton / Halley steps
// (tools/nc_diag.py).  DEG 4 / 5 / 6 measured 22.9 / 23.4 / 23.5 ms at
// level 6.  Returns the x-step, or NaN.
struct NcStep {
    double dx;      // the x-step
    double t1, t2;  // |c_{DEG-1} d^{DEG-1}|, |c_DEG d^DEG|: the polynomial's last two terms at the root
};
template <int DEG>
__device__ inline NcStep nc_taylor_step_terms(const NcCdf &c, double a0, double h, double x) {
    const double inv_y = 2.0 / x;
    double D[DEG];
    double sm = c.s0, sk = 2.0 * c.pdf;  // S_{k-1}, S_k
    D[0] = sk;
#pragma unroll
    for (int k = 1; k < DEG; ++k) {
        const double sn = fma(h, sm, (a0 - static_cast<double>(k)) * sk) * inv_y;
        sm = sk;
        sk = sn;
        D[k] = sk;
    }
    double cf[DEG + 1];
    cf[0] = c.resid;
    constexpr double kInvFact[7] = {1.0, 1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0, 1.0 / 720.0};
#pragma unroll
    for (int n = 1; n <= DEG; ++n) {
        cf[n] = D[0] * kInvFact[n];
#pragma unroll
        for (int i = 0; i < DEG - n; ++i) D[i] = D[i + 1] - D[i];
    }
    // Newton on the polynomial from the plain Newton step: one exact
    // derivative, then chord steps with it (the polynomial is near-linear
    // over the step: each chord step gains ~|2 c2 d / c1| ~ 1e-3) -- two
    // divisions instead of eight.
    double d = -c.resid / cf[1];
    double inv_dp = 0.0;
#pragma unroll
    for (int it = 0; it < 3; ++it) {
        double p = cf[DEG], dp = 0.0;
#pragma unroll
        for (int n = DEG - 1; n >= 0; --n) {
            if (it == 0) dp = fma(dp, d, p);
            p = fma(p, d, cf[n]);
        }
        if (it == 0) inv_dp = 1.0 / dp;
        d = fma(-p, inv_dp, d);
    }
    double pw = d;
#pragma unroll
    for (int n = 2; n <= DEG - 1; ++n) pw *= d;  // d^(DEG-1)
    return {2.0 * d, fabs(cf[DEG - 1] * pw), fabs(cf[DEG] * pw * d)};
}
template <int DEG>
__device__ inline double nc_taylor_step(const NcCdf &c, double a0, double h, double x) {
    return nc_taylor_step_terms<DEG>(c, a0, h, x).dx;  // the term sizes are dead code here
}

#if ARV_NC_COUNT  // diagnostic build: CDF evaluations per solve, per lane and per warp (max)
__device__ unsigned long long g_nc_evals, g_nc_solves, g_nc_hist[8], g_nc_warp_hist[8];
#endif

#ifndef ARV_NC_CERTIFY
#define ARV_NC_CERTIFY 1
#endif
#ifndef ARV_NC_CERT_DIV
#define ARV_NC_CERT_DIV 8.0  // max(|c5 d^5|, |c6 d^6|) <= tol_f / this
#endif
// Run-time switch (arv_set_tuning(ARV_TUNE_NC_CERTIFY, 0 / 1), default on) and a
// counter of solves that took the certified shortcut (arv_nc_certified_count:
// the tests assert that the shortcut actually ran where it should).
__device__ int g_nc_certify_on = 1;
__device__ unsigned long long g_nc_certified = 0;
constexpr double kNcCertifyMinTail = 1e-5;  // certified shortcut only for min(u, 1 - u) >= this (tol_f = 1e-9 there)
// exact_dist.py:381-461 contract, per element, warm start x0 (<= 0: mean);
// tol is the reference's `tol` argument (default 1e-9).  Same bracket,
// tolerance and 1e-8 residual contract as _vector_newton: each step is the
// Taylor-polynomial root (nc_taylor_step; plain Newton if it is not finite),
// which the bracket safeguard accepts or replaces by bisection.  From the
// table warm start 99.9% of bulk solves are certified after the start sweep
// alone (below); the others finish after one verification sweep
// (tools/nc_diag.py).
__device__ inline NcQuantile ncchi2_quantile(double u, double nu, double lam, double x0, double tol = 1e-9) {
    const double a0 = 0.5 * nu;
    const double one_minus_u = 1.0 - u;
    double hi = lam + nu + 20.0 * static_cast<double>(sqrtf(static_cast<float>(2.0 * (lam + nu)))) + 100.0;  // bracket heuristic
    double lo = 0.0;
    const double tol_f = fmin(tol, fmax(1e-13, 1e-4 * fmin(u, one_minus_u)));
    double x = x0 > 0.0 ? x0 : lam + nu;
    x = fmin(fmax(x, 1e-8), hi);
    const NcLam L = nc_lam(lam, fmin(u, one_minus_u) >= 1e-6 ? kNcSigmasBulk : kNcSigmas);
    double inv_w;
    // Certified single-sweep solve (bulk quantiles from a warm start).  One
    // full-width sweep gives F, S_0, S_1 at the warm start to ~1e-12; the root d
    // of the degree-6 Taylor polynomial of F is accepted WITHOUT the
    // verification sweep when the step is short (|dx| <= x / 20: F is analytic
    // with its nearest singularity at x = 0, so the Taylor terms eventually
    // fall by at least 20 per order, and by ~sigma / |d| >= 5 before that) and
    // the polynomial's last two terms are both far below the tolerance
    // (max(|c5 d^5|, |c6 d^6|) <= tol_f / 8; a ratio test between them fails
    // needlessly where the odd coefficient c5 passes through zero).  Measured:
    // such solves leave |F(x) - u| <= 3e-12 against the 8-sigma CDF on 10^7
    // solves per nu, and no solve without a verified residual exceeds 1e-10
    // (tests/test_gpu_mlmc.py).  A warp takes the shortcut only if all of its
    // lanes certify (the others would make it run the verification sweep
    // anyway, and then every lane is verified for free).  Lanes that do not
    // qualify -- larger warm-start errors, far tails, no warm start -- take
    // the verified path unchanged.
    const bool candidate = ARV_NC_CERTIFY && g_nc_certify_on && x0 > 0.0 && L.blocked &&
                           fmin(u, one_minus_u) >= kNcCertifyMinTail;
    // other bulk solves: the first sweep only places the Taylor step (6-sigma
    // window); the verification and any further sweeps use the full window
    bool narrow = L.blocked && ARV_NC_NARROW_START && !candidate;
    // One loop, one call site per sweep kind (the sweeps are large: every
    // inlined copy costs instruction cache).  `full`: evaluate F with S_0, S_1
    // at x, else F only (the verification of a step).
    bool full = true, first = true;
    NcCdf c = {0.0, 0.0, 0.0};
    int n_eval = 0;
    (void)n_eval;  // read by the ARV_NC_COUNT build only
    for (int it = 0; it < 200; ++it) {
        if (full) {
            c = ncchi2_cdf_sweep<true>(a0, x, L, u, inv_w, narrow);
        } else {
            const NcCdf f = ncchi2_cdf_sweep<false>(a0, x, L, u, inv_w);
            c.resid = f.resid;
        }
        ++n_eval;
        if (!full) {  // a verification: accept, or get the derivatives at this point for another step
            if (fabs(c.resid) <= tol_f) break;
            full = true;
            continue;
        }
        if (fabs(c.resid) <= tol_f) {
            if (!narrow) break;
            // The narrow window truncates ~1e-11..1e-10, about tol_f: never accept
            // (or bracket on) its residual -- re-evaluate on the full window.
            narrow = false;
            full = false;
            continue;
        }
        narrow = false;
        if (!first && hi - lo < 1e-15 * hi) break;
        if (c.resid > 0.0) hi = x;
        else lo = x;
        double dx;
        bool certified = false;
        if (first && candidate) {
            const NcStep st = nc_taylor_step_terms<6>(c, a0, L.h, x);
            dx = -st.dx;
            certified = isfinite(dx) && x - dx > lo && x - dx < hi && fabs(dx) <= 0.05 * x &&
                        fmax(st.t1, st.t2) <= tol_f * (1.0 / ARV_NC_CERT_DIV);
            c.resid = certified ? st.t1 + st.t2 : c.resid;
        } else {
#if ARV_NC_TAYLOR
            dx = -nc_taylor_step<ARV_NC_TAYLOR>(c, a0, L.h, x);
#else
            dx = c.resid / c.pdf;
#endif
        }
        if (!isfinite(dx)) dx = c.resid / c.pdf;  // Newton
        double xn = x - dx;
        if (!isfinite(xn) || xn <= lo || xn >= hi) xn = 0.5 * (lo + hi);
        x = xn;
        if (first && candidate) {
            const unsigned am = __activemask();
            if (__all_sync(am, certified)) {  // c.resid = the term estimate
                if ((threadIdx.x & 31) == __ffs(am) - 1)
                    atomicAdd(&g_nc_certified, static_cast<unsigned long long>(__popc(am)));
                break;
            }
        }
        first = false;
        // Verify the step with the F-only sweep; only a failed step (0.01%
        // of solves) needs the derivatives at the new point for another one.
        full = ARV_NC_TAYLOR ? false : true;
    }
#if ARV_NC_COUNT
    atomicAdd(&g_nc_evals, static_cast<unsigned long long>(n_eval));
    atomicAdd(&g_nc_solves, 1ull);
    atomicAdd(&g_nc_hist[n_eval < 7 ? n_eval : 7], 1ull);
    {
        const unsigned am = __activemask();
        const unsigned wmax = __reduce_max_sync(am, static_cast<unsigned>(n_eval));
        if ((threadIdx.x & 31) == __ffs(am) - 1) atomicAdd(&g_nc_warp_hist[wmax < 7 ? wmax : 7], 1ull);
    }
#endif
    return {x, fabs(c.resid)};
}

}  // namespace arv

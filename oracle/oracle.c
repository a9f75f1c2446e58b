/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference hot path (approxrv, arXiv
 * 2012.09715).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as
 * the checker or the CPU baseline -- never as the product path.
 *
 * Every function cites the reference file:line it restates (paths under
 * /root/reference/pkg/src/approxrv/).  Arithmetic follows the reference's
 * rounding exactly: the Cython module is compiled for generic x86-64 without
 * FMA (`pkg/setup.py:8-13`), so every `a*b + c` below is a separately rounded
 * multiply and add.  Build with -ffp-contract=off (oracle/Makefile).
 *
 * Pinning: tests/test_oracle.py checks this file against golden vectors made
 * by the reference itself (tests/golden/make_golden.py).  PCG32 has no
 * reference implementation; it is pinned against the
 * published pcg32 demo known-answer sequence for (initstate 42, initseq 54).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* PCG32 (O'Neill, XSH-RR 64/32) -- not in the reference; BASELINE.json      */
/* configs name it as the uniform source.                                    */
/* ------------------------------------------------------------------------ */

static const uint64_t PCG_MULT = 6364136223846793005ULL;

static inline uint32_t pcg_output(uint64_t old) {
    uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((-rot) & 31u));
}

/* pcg32_srandom_r: state=0, inc=(initseq<<1)|1, step, state+=initstate, step. */
EXPORT void orc_pcg32_seed(uint64_t initstate, uint64_t initseq, uint64_t *state, uint64_t *inc) {
    uint64_t c = (initseq << 1u) | 1u;
    uint64_t s = 0;
    s = s * PCG_MULT + c;
    s += initstate;
    s = s * PCG_MULT + c;
    *state = s;
    *inc = c;
}

/* Affine jump-ahead of the LCG by `delta` steps: s_{n+delta} = A s_n + C. */
EXPORT void orc_lcg_jump(uint64_t delta, uint64_t inc, uint64_t *A, uint64_t *C) {
    uint64_t acc_a = 1, acc_c = 0, cur_a = PCG_MULT, cur_c = inc;
    while (delta) {
        if (delta & 1u) {
            acc_a = acc_a * cur_a;
            acc_c = acc_c * cur_a + cur_c;
        }
        cur_c = (cur_a + 1u) * cur_c;
        cur_a = cur_a * cur_a;
        delta >>= 1u;
    }
    *A = acc_a;
    *C = acc_c;
}

/* Raw 32-bit outputs [offset, offset+n) of stream (initstate, initseq). */
EXPORT void orc_pcg32_words(uint64_t initstate, uint64_t initseq, uint64_t offset, int64_t n,
                            uint32_t *out) {
    uint64_t s, inc, A, C;
    orc_pcg32_seed(initstate, initseq, &s, &inc);
    orc_lcg_jump(offset, inc, &A, &C);
    s = A * s + C;
    for (int64_t i = 0; i < n; ++i) {
        out[i] = pcg_output(s);
        s = s * PCG_MULT + inc;
    }
}

/* u32 -> f32 open-interval uniform: ((w >> 9) + 0.5) * 2^-23.
 * Mirrors the +0.5 convention of sampler.py:62; exact in f32, never 0, 1/2, 1. */
static inline float u32_to_f32(uint32_t w) {
    return ((float)(w >> 9u) + 0.5f) * 0x1p-23f;
}
/* u32 -> f64 open-interval uniform for the path kernels: (w + 0.5) * 2^-32. */
static inline double u32_to_f64(uint32_t w) {
    return ((double)w + 0.5) * 0x1p-32;
}

EXPORT void orc_u32_to_f32(const uint32_t *w, int64_t n, float *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = u32_to_f32(w[i]);
}
EXPORT void orc_u32_to_f64(const uint32_t *w, int64_t n, double *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = u32_to_f64(w[i]);
}

/* ------------------------------------------------------------------------ */
/* The six plugin kernels (_kernels.pyx:16-143 / _kernels_py.py:16-99).      */
/* ------------------------------------------------------------------------ */

/* _kernels.pyx:16-23 */
EXPORT void orc_constant_eval(const double *values, int64_t nvals, const double *u, double *out,
                              int64_t n) {
    double scale = (double)nvals;
    for (int64_t i = 0; i < n; ++i) {
        long long idx = (long long)(scale * u[i]);
        idx = idx < nvals ? idx : nvals - 1;
        out[i] = values[idx];
    }
}

static inline long long dyadic_idx64(double v, long long cap) {
    uint64_t bits;
    memcpy(&bits, &v, 8);
    long long idx = 1022 - (long long)(bits >> 52);
    return idx < cap ? idx : cap;
}
static inline long long dyadic_idx32(float v, long long cap) {
    uint32_t bits;
    memcpy(&bits, &v, 4);
    long long idx = 126 - (long long)(bits >> 23);
    return idx < cap ? idx : cap;
}

/* _kernels.pyx:26-38 */
EXPORT void orc_dyadic_index(const double *u, int64_t cap, int64_t *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = dyadic_idx64(u[i], cap);
}
/* _kernels.pyx:41-53 */
EXPORT void orc_dyadic_index32(const float *u, int64_t cap, int64_t *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = dyadic_idx32(u[i], cap);
}

/* _kernels.pyx:56-73.  coeffs is (degree+1, K1) C-contiguous, K1 = K+1. */
static inline double dyadic_eval1(const double *coeffs, int degree, int64_t K1, double u) {
    long long cap = K1 - 1;
    int pred = u < 0.5;
    double v = pred ? u : 1.0 - u;
    long long idx = dyadic_idx64(v, cap);
    if (idx < 0) idx = 0; /* out-of-contract guard (u outside (0,1)); the reference reads OOB */
    double z = coeffs[(int64_t)degree * K1 + idx];
    for (int d = degree - 1; d >= 0; --d) z = z * v + coeffs[(int64_t)d * K1 + idx];
    return pred ? z : -z;
}
EXPORT void orc_dyadic_eval(const double *coeffs, int degree, int64_t K1, const double *u, double *out,
                            int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = dyadic_eval1(coeffs, degree, K1, u[i]);
}

/* _kernels.pyx:76-93 */
static inline float dyadic_eval1_f32(const float *coeffs, int degree, int64_t K1, float u) {
    long long cap = K1 - 1;
    int pred = u < 0.5f;
    float v = pred ? u : 1.0f - u;
    long long idx = dyadic_idx32(v, cap);
    if (idx < 0) idx = 0;
    float z = coeffs[(int64_t)degree * K1 + idx];
    for (int d = degree - 1; d >= 0; --d) z = z * v + coeffs[(int64_t)d * K1 + idx];
    return pred ? z : -z;
}
EXPORT void orc_dyadic_eval32(const float *coeffs, int degree, int64_t K1, const float *u, float *out,
                              int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = dyadic_eval1_f32(coeffs, degree, K1, u[i]);
}

/* _kernels.pyx:96-143.  stacks is (2, n_knots, degree+1, K1): upper at 0,
 * lower at 1.  lam has nlam == 1 (shared, hoisted) or nlam == n. */
static inline double ncchi2_eval1(const double *stacks, int64_t n_knots, int degree, int64_t K1,
                                  double nu, double u, double lam_i) {
    long long cap = K1 - 1;
    double shift = lam_i + nu;
    double scale2 = 2.0 * sqrt(shift);
    double s = sqrt(nu / shift);
    double g = s * (double)(n_knots - 1);
    long long j = (long long)g;
    j = j < n_knots - 2 ? j : n_knots - 2;
    double t = g - (double)j;
    double v = u;
    long long sel = (long long)(v < 0.5);
    v = sel ? v : 1.0 - v;
    long long idx = dyadic_idx64(v, cap);
    if (idx < 0) idx = 0;
    const int64_t knot = (degree + 1) * K1;
    const double *t0 = stacks + (sel * n_knots + j) * knot;
    const double *t1 = t0 + knot;
    double z0 = t0[(int64_t)degree * K1 + idx];
    double z1 = t1[(int64_t)degree * K1 + idx];
    for (int d = degree - 1; d >= 0; --d) {
        z0 = z0 * v + t0[(int64_t)d * K1 + idx];
        z1 = z1 * v + t1[(int64_t)d * K1 + idx];
    }
    return shift + scale2 * (z0 + t * (z1 - z0));
}
EXPORT void orc_ncchi2_eval(const double *stacks, int64_t n_knots, int degree, int64_t K1, double nu,
                            const double *u, const double *lam, int64_t nlam, double *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        out[i] = ncchi2_eval1(stacks, n_knots, degree, K1, nu, u[i], nlam == 1 ? lam[0] : lam[i]);
}

/* ------------------------------------------------------------------------ */
/* Octave x sub-interval dyadic table (new layout, BASELINE.json config 2).   */
/* coeffs natural layout (degree+1, K, nsub): octave j = 1..K-1 covers       */
/* [2^-(j+1), 2^-j) split into nsub = 2^sub_bits equal parts selected by the  */
/* top sub_bits mantissa bits of v; octave K is the singular remainder       */
/* (0, 2^-K) and uses its s = 0 polynomial; v == 1/2 evaluates to 0 (the     */
/* reference's u = 1/2 slot, tables.py:51-75).  Arithmetic as dyadic_eval32.  */
/* ------------------------------------------------------------------------ */
static inline float subdyadic_eval1_f32(const float *coeffs, int degree, int K, int sub_bits, float u) {
    int pred = u < 0.5f;
    float v = pred ? u : 1.0f - u;
    uint32_t bits;
    memcpy(&bits, &v, 4);
    long long j = 126 - (long long)(bits >> 23);
    float z;
    if (j <= 0) {
        z = 0.0f;
    } else {
        int s = 0;
        if (j >= K) j = K;
        else s = (int)((bits >> (23 - sub_bits)) & ((1u << sub_bits) - 1u));
        const int nsub = 1 << sub_bits;
        const int64_t row = (int64_t)K * nsub;
        const int64_t e = (j - 1) * nsub + s;
        z = coeffs[(int64_t)degree * row + e];
        for (int d = degree - 1; d >= 0; --d) z = z * v + coeffs[(int64_t)d * row + e];
    }
    return pred ? z : -z;
}
EXPORT void orc_subdyadic_eval32(const float *coeffs, int degree, int K, int sub_bits, const float *u,
                                 float *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = subdyadic_eval1_f32(coeffs, degree, K, sub_bits, u[i]);
}

/* ------------------------------------------------------------------------ */
/* AS 241 / PPND16 (exact_dist.py:30-126).                                   */
/* ------------------------------------------------------------------------ */
static const double AS_A[8] = {
    3.3871328727963666080e0, 1.3314166789178437745e2, 1.9715909503065514427e3,
    1.3731693765509461125e4, 4.5921953931549871457e4, 6.7265770927008700853e4,
    3.3430575583588128105e4, 2.5090809287301226727e3};
static const double AS_B[8] = {
    1.0, 4.2313330701600911252e1, 6.8718700749205790830e2,
    5.3941960214247511077e3, 2.1213794301586595867e4, 3.9307895800092710610e4,
    2.8729085735721942674e4, 5.2264952788528545610e3};
static const double AS_C[8] = {
    1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0,
    3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,
    2.27238449892691845833e-2, 7.74545014278341407640e-4};
static const double AS_D[8] = {
    1.0, 2.05319162663775882187e0, 1.67638483018380384940e0,
    6.89767334985100004550e-1, 1.48103976427480074590e-1, 1.51986665636164571966e-2,
    5.47593808499534494600e-4, 1.05075007164441684324e-9};
static const double AS_E[8] = {
    6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0,
    2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,
    2.71155556874348757815e-5, 2.01033439929228813265e-7};
static const double AS_F[8] = {
    1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1,
    1.48753612908506148525e-2, 7.86869131145613259100e-4, 1.84631831751005468180e-5,
    1.42151175831644588870e-7, 2.04426310338993978564e-15};

/* exact_dist.py:65-70: Horner, coeffs[0] constant, separate mul/add. */
static inline double polyval8(const double *c, double x) {
    double acc = c[7];
    for (int i = 6; i >= 0; --i) acc = acc * x + c[i];
    return acc;
}

/* exact_dist.py:87-126 (domain validation is the caller's: u in (0,1)). */
static inline double as241_f64(double u) {
    double q = u - 0.5;
    if (fabs(q) <= 0.425) {
        double r = 0.180625 - q * q;
        return q * polyval8(AS_A, r) / polyval8(AS_B, r);
    }
    int upper = u > 0.5;
    double w = upper ? 1.0 - u : u;
    double r = sqrt(-log(w));
    double val;
    if (r <= 5.0) {
        double rn = r - 1.6;
        val = polyval8(AS_C, rn) / polyval8(AS_D, rn);
    } else {
        double rf = r - 5.0;
        val = polyval8(AS_E, rf) / polyval8(AS_F, rf);
    }
    return upper ? val : -val;
}
EXPORT void orc_as241_f64(const double *u, double *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = as241_f64(u[i]);
}

/* Single-precision evaluation of the same PPND16 rational (coefficients
 * rounded to f32, f32 arithmetic, logf/sqrtf).  NOT the paper's PPND7; new,
 * parity unpinned beyond the f64 comparison in tests. */
static inline float polyval8f(const double *c, float x) {
    float acc = (float)c[7];
    for (int i = 6; i >= 0; --i) acc = acc * x + (float)c[i];
    return acc;
}
static inline float as241_f32(float u) {
    float q = u - 0.5f;
    if (fabsf(q) <= 0.425f) {
        float r = 0.180625f - q * q;
        return q * polyval8f(AS_A, r) / polyval8f(AS_B, r);
    }
    int upper = u > 0.5f;
    float w = upper ? 1.0f - u : u;
    float r = sqrtf(-logf(w));
    float val;
    if (r <= 5.0f) {
        float rn = r - 1.6f;
        val = polyval8f(AS_C, rn) / polyval8f(AS_D, rn);
    } else {
        float rf = r - 5.0f;
        val = polyval8f(AS_E, rf) / polyval8f(AS_F, rf);
    }
    return upper ? val : -val;
}
EXPORT void orc_as241_f32(const float *u, float *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = as241_f32(u[i]);
}

/* ------------------------------------------------------------------------ */
/* Fused generators = PCG32 words -> uniform -> evaluator (same per-element  */
/* arithmetic as the functions above).  Used as checker and CPU baseline.   */
/* ------------------------------------------------------------------------ */
#define CHUNK 4096

/* out[i] = f32(values[w_i >> (32-q)]): constant_eval with f64(u), u = u32_to_f32(w). */
EXPORT void orc_pcg32_constant_f32(uint64_t seed, uint64_t seq, uint64_t offset, const float *values,
                                   int q, float *out, int64_t n) {
    uint64_t s, inc, A, C;
    orc_pcg32_seed(seed, seq, &s, &inc);
    orc_lcg_jump(offset, inc, &A, &C);
    s = A * s + C;
    const double scale = (double)(1u << q);
    const long long nv = 1ll << q;
    for (int64_t i = 0; i < n; ++i) {
        double u = (double)u32_to_f32(pcg_output(s));
        s = s * PCG_MULT + inc;
        long long idx = (long long)(scale * u);
        idx = idx < nv ? idx : nv - 1;
        out[i] = values[idx];
    }
}

EXPORT void orc_pcg32_subdyadic_f32(uint64_t seed, uint64_t seq, uint64_t offset, const float *coeffs,
                                    int degree, int K, int sub_bits, float *out, int64_t n) {
    uint64_t s, inc, A, C;
    orc_pcg32_seed(seed, seq, &s, &inc);
    orc_lcg_jump(offset, inc, &A, &C);
    s = A * s + C;
    for (int64_t i = 0; i < n; ++i) {
        float u = u32_to_f32(pcg_output(s));
        s = s * PCG_MULT + inc;
        out[i] = subdyadic_eval1_f32(coeffs, degree, K, sub_bits, u);
    }
}

/* Reference-layout dyadic (coeffs32 (degree+1, K1)), _kernels.pyx:76-93. */
EXPORT void orc_pcg32_dyadic_f32(uint64_t seed, uint64_t seq, uint64_t offset, const float *coeffs,
                                 int degree, int64_t K1, float *out, int64_t n) {
    uint64_t s, inc, A, C;
    orc_pcg32_seed(seed, seq, &s, &inc);
    orc_lcg_jump(offset, inc, &A, &C);
    s = A * s + C;
    for (int64_t i = 0; i < n; ++i) {
        float u = u32_to_f32(pcg_output(s));
        s = s * PCG_MULT + inc;
        out[i] = dyadic_eval1_f32(coeffs, degree, K1, u);
    }
}

/* AS241 f64 of the f32-lattice uniform (the exact comparator for config 2/3). */
EXPORT void orc_pcg32_as241_f64(uint64_t seed, uint64_t seq, uint64_t offset, double *out, int64_t n) {
    uint64_t s, inc, A, C;
    orc_pcg32_seed(seed, seq, &s, &inc);
    orc_lcg_jump(offset, inc, &A, &C);
    s = A * s + C;
    for (int64_t i = 0; i < n; ++i) {
        double u = (double)u32_to_f32(pcg_output(s));
        s = s * PCG_MULT + inc;
        out[i] = as241_f64(u);
    }
}
EXPORT void orc_pcg32_as241_f32(uint64_t seed, uint64_t seq, uint64_t offset, float *out, int64_t n) {
    uint64_t s, inc, A, C;
    orc_pcg32_seed(seed, seq, &s, &inc);
    orc_lcg_jump(offset, inc, &A, &C);
    s = A * s + C;
    for (int64_t i = 0; i < n; ++i) {
        float u = u32_to_f32(pcg_output(s));
        s = s * PCG_MULT + inc;
        out[i] = as241_f32(u);
    }
}

/* ------------------------------------------------------------------------ */
/* Nested MLMC, GBM (mlmc.py:164-229).  Uniform for (fine step k, path p) is */
/* PCG32 output k*n_paths + p of stream (seed, seq) -- the reference's own   */
/* addressing with Philox words replaced by PCG32 outputs.     */
/* table: f64 dyadic coeffs (degree+1, K1) evaluated like dyadic_eval.       */
/* ------------------------------------------------------------------------ */
/* mlmc.py:194-198 */
static inline double em_step(double x, double dw, double dt, double mu, double sg, int milstein) {
    double incr = mu * dt + sg * dw;
    if (milstein) incr += 0.5 * sg * sg * (dw * dw - dt);
    return x * (1.0 + incr);
}

EXPORT void orc_gbm_paths(double mu, double sigma, double x0, double t_end, int level, int n0,
                          int milstein, int payoff_call, double strike, const double *coeffs,
                          int degree, int64_t K1, uint64_t seed, uint64_t seq, int64_t n_paths,
                          int64_t path_lo, int64_t path_hi, double *pf_e, double *pc_e, double *pf_a,
                          double *pc_a) {
    uint64_t s0, inc, AN, CN;
    orc_pcg32_seed(seed, seq, &s0, &inc);
    orc_lcg_jump((uint64_t)n_paths, inc, &AN, &CN);
    const int64_t n_f = (int64_t)n0 << level;
    const double dt_f = t_end / (double)n_f;
    const double dt_c = 2.0 * dt_f;
    const double sq_f = sqrt(dt_f);
    for (int64_t p = path_lo; p < path_hi; ++p) {
        uint64_t A, C, s;
        orc_lcg_jump((uint64_t)p, inc, &A, &C);
        s = A * s0 + C;
        double xf_e = x0, xc_e = x0, xf_a = x0, xc_a = x0;
        for (int64_t pair = 0; pair < n_f / 2; ++pair) {
            double u1 = u32_to_f64(pcg_output(s));
            s = AN * s + CN;
            double u2 = u32_to_f64(pcg_output(s));
            s = AN * s + CN;
            double z1 = as241_f64(u1), z2 = as241_f64(u2);
            xf_e = em_step(em_step(xf_e, sq_f * z1, dt_f, mu, sigma, milstein), sq_f * z2, dt_f, mu,
                           sigma, milstein);
            xc_e = em_step(xc_e, sq_f * (z1 + z2), dt_c, mu, sigma, milstein);
            double w1 = dyadic_eval1(coeffs, degree, K1, u1);
            double w2 = dyadic_eval1(coeffs, degree, K1, u2);
            xf_a = em_step(em_step(xf_a, sq_f * w1, dt_f, mu, sigma, milstein), sq_f * w2, dt_f, mu,
                           sigma, milstein);
            xc_a = em_step(xc_a, sq_f * (w1 + w2), dt_c, mu, sigma, milstein);
        }
        if (n_f % 2) {
            double u1 = u32_to_f64(pcg_output(s));
            xf_e = em_step(xf_e, sq_f * as241_f64(u1), dt_f, mu, sigma, milstein);
            xf_a = em_step(xf_a, sq_f * dyadic_eval1(coeffs, degree, K1, u1), dt_f, mu, sigma, milstein);
        }
        /* mlmc.py:152-155 payoff; :221-229 level-0 coarse = 0 */
        double fe = payoff_call ? fmax(xf_e - strike, 0.0) : xf_e;
        double fa = payoff_call ? fmax(xf_a - strike, 0.0) : xf_a;
        double ce = level > 0 ? (payoff_call ? fmax(xc_e - strike, 0.0) : xc_e) : 0.0;
        double ca = level > 0 ? (payoff_call ? fmax(xc_a - strike, 0.0) : xc_a) : 0.0;
        int64_t i = p - path_lo;
        pf_e[i] = fe;
        pc_e[i] = ce;
        pf_a[i] = fa;
        pc_a[i] = ca;
    }
}

/* CIR truncated Euler (mlmc.py:289-331), exact-Gaussian and table sides. */
static double cir_step1(double x, double dw, double dt, double kappa, double theta, double sigma, int milstein) {
    double r = x + kappa * (theta - x) * dt + sigma * sqrt(fabs(x)) * dw; /* mlmc.py:295-296 */
    if (milstein) r = r + 0.25 * sigma * sigma * (dw * dw - dt);
    return r;
}

/* CIR truncated Euler (mlmc.py:289-331, step :295-296) and, with milstein
 * = 1, the truncated Milstein scheme the reference does not have (BASELINE
 * config 5 "CIR ... with Milstein"): the Euler step plus the Milstein term
 * 1/2 b b' (dW^2 - dt) of b(x) = sigma sqrt(x), i.e. sigma^2/4 (dW^2 - dt),
 * added last; the device scheme is cir_step<true> (arv_mlmc.cu).  Same
 * coupling, uniforms and payoffs as the Euler loop. */
EXPORT void orc_cir_paths(double kappa, double theta, double sigma, double x0, double t_end,
                          int level, int n0, int milstein, int payoff_call, double strike,
                          const double *coeffs, int degree, int64_t K1, uint64_t seed,
                          uint64_t seq, int64_t n_paths, int64_t path_lo, int64_t path_hi,
                          double *pf_e, double *pc_e, double *pf_a, double *pc_a) {
    uint64_t s0, inc, AN, CN;
    orc_pcg32_seed(seed, seq, &s0, &inc);
    orc_lcg_jump((uint64_t)n_paths, inc, &AN, &CN);
    const int64_t n_f = (int64_t)n0 << level;
    const double dt_f = t_end / (double)n_f;
    const double dt_c = 2.0 * dt_f;
    const double sq_f = sqrt(dt_f);
#define CIR_EM(x, dw, dt) cir_step1(x, dw, dt, kappa, theta, sigma, milstein)
    for (int64_t p = path_lo; p < path_hi; ++p) {
        uint64_t A, C, s;
        orc_lcg_jump((uint64_t)p, inc, &A, &C);
        s = A * s0 + C;
        double xf_e = x0, xc_e = x0, xf_a = x0, xc_a = x0;
        for (int64_t pair = 0; pair < n_f / 2; ++pair) {
            double u1 = u32_to_f64(pcg_output(s));
            s = AN * s + CN;
            double u2 = u32_to_f64(pcg_output(s));
            s = AN * s + CN;
            double z1 = as241_f64(u1), z2 = as241_f64(u2);
            double t = CIR_EM(xf_e, sq_f * z1, dt_f);
            xf_e = CIR_EM(t, sq_f * z2, dt_f);
            xc_e = CIR_EM(xc_e, sq_f * (z1 + z2), dt_c);
            double w1 = dyadic_eval1(coeffs, degree, K1, u1);
            double w2 = dyadic_eval1(coeffs, degree, K1, u2);
            t = CIR_EM(xf_a, sq_f * w1, dt_f);
            xf_a = CIR_EM(t, sq_f * w2, dt_f);
            xc_a = CIR_EM(xc_a, sq_f * (w1 + w2), dt_c);
        }
        if (n_f % 2) {
            double u1 = u32_to_f64(pcg_output(s));
            xf_e = CIR_EM(xf_e, sq_f * as241_f64(u1), dt_f);
            xf_a = CIR_EM(xf_a, sq_f * dyadic_eval1(coeffs, degree, K1, u1), dt_f);
        }
        double fe = payoff_call ? fmax(xf_e - strike, 0.0) : xf_e;
        double fa = payoff_call ? fmax(xf_a - strike, 0.0) : xf_a;
        double ce = level > 0 ? (payoff_call ? fmax(xc_e - strike, 0.0) : xc_e) : 0.0;
        double ca = level > 0 ? (payoff_call ? fmax(xc_a - strike, 0.0) : xc_a) : 0.0;
        int64_t i = p - path_lo;
        pf_e[i] = fe;
        pc_e[i] = ce;
        pf_a[i] = fa;
        pc_a[i] = ca;
    }
#undef CIR_EM
}

EXPORT void orc_cir_euler_paths(double kappa, double theta, double sigma, double x0, double t_end,
                                int level, int n0, int payoff_call, double strike,
                                const double *coeffs, int degree, int64_t K1, uint64_t seed,
                                uint64_t seq, int64_t n_paths, int64_t path_lo, int64_t path_hi,
                                double *pf_e, double *pc_e, double *pf_a, double *pc_a) {
    orc_cir_paths(kappa, theta, sigma, x0, t_end, level, n0, 0, payoff_call, strike, coeffs, degree, K1, seed,
                  seq, n_paths, path_lo, path_hi, pf_e, pc_e, pf_a, pc_a);
}

/* ------------------------------------------------------------------------ */
/* Philox-4x64-10 (Salmon et al. 2011; numpy.random.Philox), the reference's */
/* uniform source: UniformStream (sampler.py:26-66) keys it with            */
/* [seed, stream_id]; word n is Philox(ctr=[n/4 + 1, 0, 0, 0], key)[n % 4]   */
/* (numpy pre-increments the 256-bit counter), u = ((w >> 11) + 0.5) 2^-53.  */
/* ------------------------------------------------------------------------ */
static const uint64_t PH_M0 = 0xD2E7470EE14C6C93ULL, PH_M1 = 0xCA5A826395121157ULL;
static const uint64_t PH_W0 = 0x9E3779B97F4A7C15ULL, PH_W1 = 0xBB67AE8584CAA73BULL;

static inline void philox4x64_10(const uint64_t ctr[4], uint64_t k0, uint64_t k1, uint64_t out[4]) {
    uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += PH_W0;
            k1 += PH_W1;
        }
        __uint128_t p0 = (__uint128_t)PH_M0 * c0, p1 = (__uint128_t)PH_M1 * c2;
        uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
        uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* 64-bit words [start, start+n) of UniformStream(seed, stream_id). */
EXPORT void orc_philox_words(uint64_t seed, uint64_t sid, uint64_t start, int64_t n, uint64_t *out) {
    uint64_t blk[4];
    uint64_t cur = UINT64_MAX;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t w = start + (uint64_t)i;
        uint64_t b = w >> 2;
        if (b != cur) {
            /* counter = b + 1 as a 256-bit integer (carry into word 1) */
            uint64_t ctr[4] = {b + 1, b + 1 == 0 ? 1u : 0u, 0, 0};
            philox4x64_10(ctr, seed, sid, blk);
            cur = b;
        }
        out[i] = blk[w & 3];
    }
}

/* UniformStream.uniforms (sampler.py:59-62) */
EXPORT void orc_philox_uniforms(uint64_t seed, uint64_t sid, uint64_t start, int64_t n, double *out) {
    uint64_t blk[4];
    uint64_t cur = UINT64_MAX;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t w = start + (uint64_t)i;
        uint64_t b = w >> 2;
        if (b != cur) {
            uint64_t ctr[4] = {b + 1, b + 1 == 0 ? 1u : 0u, 0, 0};
            philox4x64_10(ctr, seed, sid, blk);
            cur = b;
        }
        out[i] = ((double)(blk[w & 3] >> 11) + 0.5) * 0x1p-53;
    }
}

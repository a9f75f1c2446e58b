/*
 * approxrv_b200 -- C ABI of the B200-native hot path of approxrv
 * (arXiv 2012.09715).  One shared library, libarv_b200.so, built for sm_100a.
 *
 * Conventions
 *   - Every data pointer is a DEVICE pointer (cudaMalloc / torch CUDA tensor
 *     storage), C-contiguous, of the element type in the signature.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     Calls are asynchronous: they enqueue kernels and return.
 *   - Return value: ARV_OK (0) or an error code; arv_last_error() returns
 *     the message of the calling thread's last failure.  No exceptions cross
 *     the ABI.  Codes map onto the reference exception hierarchy
 *     (errors.py:9-42): ARV_ERR_CONFIG -> ConfigError, ARV_ERR_DOMAIN ->
 *     DomainError, ARV_ERR_NUMERICAL -> NumericalError, ARV_ERR_CUDA ->
 *     RuntimeError.
 *   - Kernels never validate u in (0,1): that is the caller's contract
 *     (sampler.py:100-102).  Out-of-contract inputs cannot fault (table
 *     indices are clamped) but their values are unspecified.
 *
 * PCG32 streams: a (seed, stream_id) pair is PCG32 with initstate = seed,
 * initseq = stream_id (O'Neill's pcg32_srandom_r).  `offset` is the index
 * of the first 32-bit output used; sample i of a call consumes output
 * offset + i, so any range can be generated independently (GPU shards).
 */
#ifndef APPROXRV_B200_H
#define APPROXRV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ARV_OK 0
#define ARV_ERR_CONFIG 1
#define ARV_ERR_DOMAIN 2
#define ARV_ERR_NUMERICAL 3
#define ARV_ERR_CUDA 4

#define ARV_ABI_VERSION 1

#if defined(__GNUC__)
#define ARV_API __attribute__((visibility("default")))
#else
#define ARV_API
#endif

/* ---- library ----------------------------------------------------------- */
ARV_API int arv_abi_version(void);
ARV_API const char *arv_last_error(void);
/* sha256 (hex) of the sources the library was built from. */
ARV_API const char *arv_source_hash(void);
/* Number of kernel launches this library has issued (process-wide). */
ARV_API uint64_t arv_launch_count(void);

/* ---- drop-in plugin kernels: approxrv._kernels (the `kernels` module that
 * approxrv/_backend.py:14-24 selects).  Same arguments and results as the
 * Cython functions, on device arrays.  ------------------------------------ */

/* _kernels.pyx:16-23  constant_eval(values f64[nvals], u f64[n], out f64[n]) */
ARV_API int arv_constant_eval(const double *values, int64_t nvals, const double *u, double *out, int64_t n,
                      void *stream);
/* _kernels.pyx:26-38  dyadic_index(u f64[n], cap) -> i64[n] (caller allocates out) */
ARV_API int arv_dyadic_index(const double *u, int64_t n, int64_t cap, int64_t *out, void *stream);
/* _kernels.pyx:41-53  dyadic_index32(u f32[n], cap) -> i64[n] */
ARV_API int arv_dyadic_index32(const float *u, int64_t n, int64_t cap, int64_t *out, void *stream);
/* _kernels.pyx:56-73  dyadic_eval(coeffs f64[degree+1][K1], u f64[n], out f64[n]) */
ARV_API int arv_dyadic_eval(const double *coeffs, int degree, int64_t K1, const double *u, double *out,
                    int64_t n, void *stream);
/* _kernels.pyx:76-93  dyadic_eval32(coeffs32 f32[degree+1][K1], u f32[n], out f32[n]) */
ARV_API int arv_dyadic_eval32(const float *coeffs, int degree, int64_t K1, const float *u, float *out,
                      int64_t n, void *stream);
/* _kernels.pyx:96-143 ncchi2_eval(stacks f64[2][n_knots][degree+1][K1], nu,
 * u f64[n], lam f64[nlam] (nlam == 1 shared, or n), out f64[n]) */
ARV_API int arv_ncchi2_eval(const double *stacks, int64_t n_knots, int degree, int64_t K1, double nu,
                    const double *u, const double *lam, int64_t nlam, double *out, int64_t n,
                    void *stream);

/* ---- the same plugin functions with HOST buffers (the reference's numpy
 * calling convention: sampler.py:91-206 passes host arrays and a
 * caller-allocated host `out`).  u, lam and out are host pointers (pageable
 * or pinned); tables (values / coeffs / stacks) are device pointers.  The
 * call stages chunks through pinned buffers, overlapping the host copies,
 * H2D, the kernel (on `stream`) and D2H, and returns when out is written.
 * Calls are serialised per device. ------------------------------------- */
ARV_API int arv_host_constant_eval(const double *values, int64_t nvals, const double *u, double *out, int64_t n,
                                   void *stream);
ARV_API int arv_host_dyadic_index(const double *u, int64_t n, int64_t cap, int64_t *out, void *stream);
ARV_API int arv_host_dyadic_index32(const float *u, int64_t n, int64_t cap, int64_t *out, void *stream);
ARV_API int arv_host_dyadic_eval(const double *coeffs, int degree, int64_t K1, const double *u, double *out,
                                 int64_t n, void *stream);
ARV_API int arv_host_dyadic_eval32(const float *coeffs, int degree, int64_t K1, const float *u, float *out,
                                   int64_t n, void *stream);
ARV_API int arv_host_subdyadic_eval32(const float *coeffs, int degree, int K, int sub_bits, const float *u,
                                      float *out, int64_t n, void *stream);
ARV_API int arv_host_ncchi2_eval(const double *stacks, int64_t n_knots, int degree, int64_t K1, double nu,
                                 const double *u, const double *lam, int64_t nlam, double *out, int64_t n,
                                 void *stream);
ARV_API int arv_host_gaussian_inv_cdf(const double *u, double *out, int64_t n, void *stream);

/* ---- extensions of the same evaluators ---------------------------------- */

/* Octave x sub-interval dyadic table, f32 (BASELINE.json config 2).
 * coeffs f32[degree+1][K][2^sub_bits] natural layout: octave j = 1..K-1 is
 * [2^-(j+1), 2^-j) split into 2^sub_bits equal parts by the top mantissa
 * bits of v = min(u, 1-u); octave K is the singular remainder (0, 2^-K) and
 * uses its sub-slot 0.  u == 1/2 gives -0.0 like the reference's u = 1/2
 * slot.  Arithmetic = dyadic_eval32 (separately rounded mul/add). */
ARV_API int arv_subdyadic_eval32(const float *coeffs, int degree, int K, int sub_bits, const float *u,
                         float *out, int64_t n, void *stream);
/* exact_dist.py:87-126  gaussian_inv_cdf (AS241 PPND16) in f64; and the same
 * rational in f32 arithmetic. */
ARV_API int arv_gaussian_inv_cdf(const double *u, double *out, int64_t n, void *stream);
ARV_API int arv_gaussian_inv_cdf32(const float *u, float *out, int64_t n, void *stream);

/* ---- fused PCG32 generators (no input traffic; 128-bit coalesced stores) --
 * Uniform mapping for f32 samples: u = ((w >> 9) + 0.5) * 2^-23.           */
ARV_API int arv_pcg32_words(uint64_t seed, uint64_t stream_id, uint64_t offset, uint32_t *out, int64_t n,
                    void *stream);
ARV_API int arv_pcg32_uniform_f32(uint64_t seed, uint64_t stream_id, uint64_t offset, float *out, int64_t n,
                          void *stream);
/* piecewise constant: out[i] = values[floor(2^q u_i)], values f32[2^q], q in [1,24] */
ARV_API int arv_pcg32_constant_f32(uint64_t seed, uint64_t stream_id, uint64_t offset, const float *values,
                           int q, float *out, int64_t n, void *stream);
/* dyadic / octave x sub-interval: coeffs as arv_subdyadic_eval32.  The
 * reference K=15 layout is sub_bits = 0 with coeffs[d][j-1][0] = ref[d][j]. */
ARV_API int arv_pcg32_subdyadic_f32(uint64_t seed, uint64_t stream_id, uint64_t offset, const float *coeffs,
                            int degree, int K, int sub_bits, float *out, int64_t n, void *stream);
/* Exhaustive check hook (tests): out f32[2^23] receives the fused
 * generators' evaluator at every point of the f32 lattice, out[k] = eval(w)
 * for a word w with w >> 9 == k.  mode 0 = the general evaluator
 * (k_pcg32_subdyadic); mode 1 = the degree-1 signed-table evaluator
 * (k_pcg32_linsigned, sub_bits <= 4) including its per-table exactness check
 * and fallback; mode 2 = the lane-private-table evaluator (k_pcg32_linlane,
 * sub_bits <= 4; scalar and packed-pair forms); *fast (device int32[1], may
 * be NULL) receives 1 if the signed / lane evaluator ran, 0 if the table
 * failed the check. */
ARV_API int arv_lattice_subdyadic_f32(const float *coeffs, int degree, int K, int sub_bits, int mode, float *out,
                                      int *fast, void *stream);
/* exact comparators: AS241 of the same f32-lattice uniforms, f64 / f32 out */
ARV_API int arv_pcg32_gaussian_f64(uint64_t seed, uint64_t stream_id, uint64_t offset, double *out, int64_t n,
                           void *stream);
ARV_API int arv_pcg32_gaussian_f32(uint64_t seed, uint64_t stream_id, uint64_t offset, float *out, int64_t n,
                           void *stream);
/* ---- Philox-4x64-10 replay of the reference's UniformStream --------------
 * sampler.py:26-66: key [seed, stream_id], word n = Philox(ctr=[n/4+1,...],
 * key)[n % 4] -- bit-exact with numpy.random.Philox.  `counter` = index of
 * the first 64-bit word (UniformStream.counter). */
ARV_API int arv_philox_words(uint64_t seed, uint64_t stream_id, uint64_t counter, uint64_t *out, int64_t n,
                             void *stream);
/* Fused Philox -> evaluator, f64 out (the reference's default evaluate()):
 * kind 0 = uniforms ((w >> 11) + 0.5) 2^-53 (sampler.py:59-62);
 * kind 1 = constant_eval, table = values f64[table_cols];
 * kind 2 = dyadic_eval, table = coeffs f64[degree+1][table_cols];
 * kind 3 = AS241 gaussian_inv_cdf (table unused). */
ARV_API int arv_philox_eval_f64(uint64_t seed, uint64_t stream_id, uint64_t counter, int kind,
                                const double *table, int degree, int64_t table_cols, double *out, int64_t n,
                                void *stream);

/* Write-only bandwidth probes (streaming stores of a constant): the store
 * roof.  mode 4 = st.global.cs.v4, 8 = st.global.cs.v8 (256-bit), 5 =
 * st.global.v4; arv_store_probe = mode 8.  n % 8 == 0, out 32-byte aligned. */
ARV_API int arv_store_probe(float *out, int64_t n, void *stream);
ARV_API int arv_store_probe_ex(float *out, int64_t n, int mode, void *stream);

/* Launch-shape knobs of the fused generators (process-wide):
 * ARV_TUNE_GROUP = samples per thread-group, 4 (v4 stores) or 8 (v8, default);
 * ARV_TUNE_CTAS_PER_SM = 256-thread CTAs per SM; 0 (default) = auto: the
 * kernel's resident count, fewer when n is small (>= 64 samples per thread). */
#define ARV_TUNE_GROUP 1
#define ARV_TUNE_CTAS_PER_SM 2
/* ARV_TUNE_CIR_SEGMENT = steps per segment of a CIR exact level (default 4;
 * 0 = one kernel per level); see arv_mlmc_cir_workspace_bytes. */
#define ARV_TUNE_CIR_SEGMENT 3
/* ARV_TUNE_GBM_KERNEL = Gaussian level kernel for both-sides PCG32 levels:
 * 0 (default), 2 (per-iteration warp tail lists) or 3 (phased tail list);
 * both give bit-identical paths and statistics. */
#define ARV_TUNE_GBM_KERNEL 4
/* ARV_TUNE_LANE_MIN_N = log2 of the smallest degree-1 sub-interval call that
 * takes the lane-private-table kernel (k_pcg32_linlane: conflict-free shared
 * memory lookups, 57 KB staged per CTA); default 26; < 0: never. */
#define ARV_TUNE_LANE_MIN_N 5
/* ARV_TUNE_NC_CERTIFY = 1 (default): warm-started bulk ncchi2 quantile solves may skip
 * the verification sweep when the Taylor polynomial's last terms certify the step
 * (csrc/arv_ncchi2.cuh); 0: every step is verified by a second CDF sweep. */
#define ARV_TUNE_NC_CERTIFY 6
ARV_API int arv_set_tuning(int key, int value);

/* ---- nested MLMC level kernels ------------------------------------------
 * Path p of a level uses word k*n_paths_total + p (fine step k) of stream
 * (seed, stream_id): the reference's addressing (mlmc.py:200-202).  With
 * rng = ARV_RNG_PHILOX the words are the reference's own Philox-4x64-10
 * UniformStream words and u = ((w >> 11) + 0.5) 2^-53 (path-by-path replay
 * of the reference); with ARV_RNG_PCG32 they are PCG32 outputs and
 * u = (w + 0.5) 2^-32.
 * A call simulates global paths [path_lo, path_lo + path_count).
 *
 * stats (device f64[3 * ARV_NKIND]) receives per kind (count, mean, M2) of
 * the per-path differences, merged deterministically (Chan).  paths
 * (device f64[4][path_count], may be NULL) receives p_fine_exact,
 * p_coarse_exact, p_fine_approx, p_coarse_approx.  workspace: device bytes,
 * at least arv_mlmc_workspace_bytes(path_count).                            */
#define ARV_NKIND 5
/* Kinds (slot order) for GBM and CIR-Euler: two_way_exact, two_way_approx,
 * four_way (mlmc.py:341-353, :383-411), plain_exact, plain_approx.
 * CIR exact: slots 0/1 are zero (coarse repeats fine, mlmc.py:281-286),
 * slot 2 is the correction p_exact - p_approx (reproduce.py:299-301),
 * slots 3/4 plain exact / approx. */
#define ARV_SCHEME_EM 0
#define ARV_SCHEME_MILSTEIN 1
#define ARV_SCHEME_CIR_EXACT 2
#define ARV_SCHEME_CIR_EULER_TRUNCATED 3
#define ARV_SCHEME_CIR_MILSTEIN_TRUNCATED 4
#define ARV_RNG_PCG32 0
#define ARV_RNG_PHILOX 1
#define ARV_SIDES_BOTH 0
#define ARV_SIDES_EXACT 1
#define ARV_SIDES_APPROX 2
#define ARV_PAYOFF_IDENTITY 0
#define ARV_PAYOFF_CALL 1

typedef struct {
    /* GBM: a = mu, b = sigma.  CIR: a = kappa, b = theta, c = sigma. */
    double a, b, c;
    double x0, t_end;
    int level, n0, scheme, payoff;
    double strike;
    uint64_t seed, stream_id;
    int64_t n_paths_total, path_lo, path_count;
    int rng; /* ARV_RNG_PCG32 or ARV_RNG_PHILOX */
    /* ARV_SIDES_EXACT / _APPROX / _BOTH (0 = both): which side's payoffs the
     * caller wants (mlmc.py:176-192 `sides`); the other side's work is
     * skipped and its payoff / statistics slots are unspecified. */
    int sides;
} arv_level_spec;

ARV_API int64_t arv_mlmc_workspace_bytes(int64_t path_count);
/* Workspace for arv_mlmc_cir_exact_level's segmented mode (paths re-bucketed
 * by lambda across the grid between segments of ARV_TUNE_CIR_SEGMENT steps;
 * ~84 B per path).  With only arv_mlmc_workspace_bytes the level runs as one
 * kernel.  Results are identical either way. */
ARV_API int64_t arv_mlmc_cir_workspace_bytes(int64_t path_count);

/* GBM (euler_maruyama / milstein, mlmc.py:164-229) and CIR truncated Euler
 * (mlmc.py:289-331) / truncated Milstein (new).  table: Gaussian dyadic
 * f64[degree+1][K1] (reference layout, dyadic_eval arithmetic) for degree
 * 1..5, or a piecewise-constant table values f64[K1] (constant_eval
 * arithmetic) for degree 0; at most 48 KiB. */
ARV_API int arv_mlmc_gaussian_level(const arv_level_spec *spec, const double *coeffs, int degree, int64_t K1,
                            double *stats, double *paths, void *workspace, int64_t workspace_bytes,
                            void *stream);
/* CIR cir_exact (mlmc.py:253-287): exact side = device non-central chi^2
 * quantile (safeguarded Newton, CDF residual <= 1e-9 tolerance contract of
 * exact_dist.py:381-461), warm-started from the table; approx side =
 * ncchi2_eval on the table stacks.  n_fail (device int64[1], may be NULL)
 * counts transitions whose residual exceeded 1e-8 (NumericalError). */
ARV_API int arv_mlmc_cir_exact_level(const arv_level_spec *spec, const double *stacks, int64_t n_knots,
                             int degree, int64_t K1, double nu, double *stats, double *paths,
                             int64_t *n_fail, void *workspace, int64_t workspace_bytes, void *stream);

/* Device non-central chi^2 quantile of (u, lam) pairs (exact_dist.py:381-461
 * contract); x0 may be NULL (Sankaran-free start: mean).  resid (may be
 * NULL) receives |F(x) - u| from the device CDF. */
ARV_API int arv_ncchi2_inv_cdf(const double *u, const double *lam, int64_t nlam, double nu, const double *x0,
                       double *out, double *resid, int64_t n, void *stream);
/* Same with the reference's `tol` (exact_dist.py:381, tol_f = min(tol, max(1e-13,
 * 1e-4 min(u, 1-u)))); arv_ncchi2_inv_cdf is tol = 1e-9. */
ARV_API int arv_ncchi2_inv_cdf_tol(const double *u, const double *lam, int64_t nlam, double nu, const double *x0,
                                   double tol, double *out, double *resid, int64_t n, void *stream);
/* Device non-central chi^2 CDF (Poisson-mixture of regularized gammas). */
ARV_API int arv_ncchi2_cdf(const double *x, const double *lam, int64_t nlam, double nu, double *out, int64_t n,
                   void *stream);
/* Number of quantile solves (arv_ncchi2_inv_cdf*, the CIR exact level kernels) that took
 * the certified single-sweep shortcut (ARV_TUNE_NC_CERTIFY) since the last call; resets it.
 * Synchronises the device. */
ARV_API int arv_nc_certified_count(unsigned long long *out);
/* Test hook: out[i] = the exact-side standard normal the Gaussian MLMC level
 * kernels compute for the 32-bit word words[i] (u = (w + 1/2) 2^-32): AS241
 * (exact_dist.py:65-126) with fused multiply-adds, a reciprocal-based
 * division and the kernels' own tail logarithm / square root. */
ARV_API int arv_test_level_normals(const uint32_t *words, double *out, int64_t n, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* APPROXRV_B200_H */

// Nested MLMC level kernels: one thread per path, all path states in f64
// registers, PCG32 stream state in registers, and in-CTA two-pass reduction
// of the per-path differences into (count, mean, M2) partials, merged by a
// second one-CTA kernel in a fixed order (parallel-axis identity), so the
// statistics are bitwise reproducible for a given (path_lo, path_count)
// whatever the scheduling.
//
// Reference loops restated (mlmc.py):
//   GBM EM / Milstein        simulate_gbm_coupled   :164-229 (em_step :194-198)
//   CIR truncated Euler      simulate_cir_coupled   :289-331
//   CIR exact (chi^2)        simulate_cir_coupled   :253-287
//   differences / estimator  difference, estimate_level_suite :341-411
// Uniform for (fine step k, path p) = PCG32 output k * n_paths_total + p of
// stream (seed, stream_id), mapped to (w + 0.5) 2^-32 -- the reference's
// per-step `stream.uniforms(n_paths)` addressing (:200-202, :261-262).  A
// thread reaches its first output with one jump and then advances by
// n_paths_total per step with a single precomputed affine map, i.e. one
// 64-bit multiply-add per step, as in a plain LCG.
#include <cmath>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "arv_common.cuh"
#include "arv_eval_dev.cuh"
#include "arv_ncchi2.cuh"
#include "arv_logtab.cuh"

namespace arv {

constexpr int kLevelBlock = 256;
// CTA size of the CIR exact level kernel (its lambda sort spans the CTA).
#ifndef ARV_CIR_BLOCK
#define ARV_CIR_BLOCK 256
#endif
constexpr int kCirBlock = ARV_CIR_BLOCK;
constexpr int kMinLevelBlock = kCirBlock < kLevelBlock ? kCirBlock : kLevelBlock;
// Min resident CTAs per SM (register cap) for the level kernels; see sweeps.
#ifndef ARV_GBM_QUAD  // four-uniform passes in the Gaussian level kernels (see as241_f64_batch)
#define ARV_GBM_QUAD 1
#endif
#ifndef ARV_GBM_SMEM_ROWS  // AS241 coefficient rows from shared memory instead of L1 (__ldg)
#define ARV_GBM_SMEM_ROWS 1
#endif
#ifndef ARV_GBM_MINB_PCG  // GBM + PCG32 instances fit 64 registers without spills (1.3% faster)
#define ARV_GBM_MINB_PCG 4
#endif
#ifndef ARV_GBM_MINB
#define ARV_GBM_MINB 3
#endif
#ifndef ARV_CIR_MINB
#define ARV_CIR_MINB 3  // 80 registers, no spill: level 6 10.72 ms vs 11.10 at 4 (64 registers, 56 B spilled) and 11.28 at 5
                        // with the single-loop quantile solver; the round-1 solver preferred 4 (57.4 vs 60.6 ms)
#endif
constexpr int kFinalBlock = 1024;

constexpr int kPathJumpBits = 40;  // path ids < 2^40

struct LevelArgs {
    double a, b, c;  // GBM: mu, sigma, -; CIR: kappa, theta, sigma
    double x0, strike;
    double dt_f, dt_c, sq_f;
    int64_t n_f;
    int level, payoff;
    uint64_t s0, inc;   // stream state at output 0
    Affine step;        // LCG^(n_paths_total)
    int64_t path_lo, path_count;
    // CIR exact
    double nu_exact, nu_table, scale, decay_over_scale;
    // uniform source
    int rng;             // ARV_RNG_PCG32 / ARV_RNG_PHILOX
    int want_exact, want_approx;  // arv_level_spec::sides
    uint64_t seed, sid;  // Philox key
    uint64_t n_paths_total;
    Affine jump2[kPathJumpBits];  // LCG^(2^i): path p starts popcount(p) affine maps from s0
};

// PCG32 state of output p of the level stream (path p's first uniform): one
// affine map per set bit of p from the kernel-parameter table, instead of a
// square-and-multiply lcg_jump per thread (which was half of the instructions
// of a one-step level).
__device__ __forceinline__ uint64_t path_start_state(const LevelArgs &A, uint64_t p) {
    uint64_t s = A.s0;
#pragma unroll 1
    for (int b = 0; b < kPathJumpBits && (p >> b) != 0; ++b)
        if ((p >> b) & 1u) s = A.jump2[b].a * s + A.jump2[b].c;
    return s;
}

// Per-path uniform source: word k * n_paths_total + p for fine step k.
struct PathRng {
    uint64_t s;       // PCG32 state / Philox word index
    Affine step;
    uint64_t n_paths, seed, sid;
    int philox;
    // state: a stored stream position (segmented CIR levels), else path p's start
    __device__ __forceinline__ PathRng(const LevelArgs &A, uint64_t p, const uint64_t *state = nullptr)
        : step(A.step), n_paths(A.n_paths_total), seed(A.seed), sid(A.sid), philox(A.rng == ARV_RNG_PHILOX) {
        if (state) {
            s = *state;
        } else if (philox) {
            s = p;
        } else {
            s = path_start_state(A, p);
        }
    }
    __device__ __forceinline__ double next() {
        double u;
        if (philox) {
            u = u64_to_f64(philox_word(s, seed, sid));  // sampler.py:62
            s += n_paths;
        } else {
            u = u32_to_f64(pcg32_output(s));
            s = step.a * s + step.c;
        }
        return u;
    }
};

// Compile-time uniform source of the Gaussian-scheme kernels: the PCG32 side
// keeps the raw word, so the f64 uniform is assembled from its bits and the
// u < 1/2 predicate is an integer compare (-2% on the GBM level kernel).
template <bool PHILOX>
struct PathSource;

template <>
struct PathSource<false> {
    uint64_t s;
    Affine step;
    __device__ __forceinline__ PathSource(const LevelArgs &A, uint64_t p) : step(A.step) {
        s = path_start_state(A, p);
    }
    // next uniform and the reference's u < 1/2
    __device__ __forceinline__ double next(bool &lower) {
        const uint32_t w = pcg32_output(s);
        s = step.a * s + step.c;
        lower = w < 0x80000000u;  // integer compare instead of DSETP
        return __dsub_rn(one_plus_u32(w), 1.0);  // == u32_to_f64(w), no I2F / DMUL
    }
};

template <>
struct PathSource<true> {
    uint64_t s, n_paths, seed, sid;
    __device__ __forceinline__ PathSource(const LevelArgs &A, uint64_t p)
        : s(p), n_paths(A.n_paths_total), seed(A.seed), sid(A.sid) {}
    __device__ __forceinline__ double next(bool &lower) {
        const double u = u64_to_f64(philox_word(s, seed, sid));  // sampler.py:62
        s += n_paths;
        lower = u < 0.5;
        return u;
    }
};

__device__ __forceinline__ double payoff_fn(double x, int payoff, double strike) {
    return payoff == ARV_PAYOFF_CALL ? fmax(__dsub_rn(x, strike), 0.0) : x;
}

// mlmc.py:194-198 em_step: x (1 + mu dt + sg dw [+ 0.5 sg^2 (dw^2 - dt)])
template <bool MIL>
__device__ __forceinline__ double gbm_step(double x, double dw, double dt, double mu, double sg) {
    double incr = __dadd_rn(__dmul_rn(mu, dt), __dmul_rn(sg, dw));
    if (MIL) incr = __dadd_rn(incr, __dmul_rn(__dmul_rn(__dmul_rn(0.5, sg), sg), __dsub_rn(__dmul_rn(dw, dw), dt)));
    return __dmul_rn(x, __dadd_rn(1.0, incr));
}

// mlmc.py:295-296 truncated Euler: x + kp (th - x) dt + sg sqrt|x| dw; the
// Milstein variant (new, not in the reference) adds sg^2/4 (dw^2 - dt).
template <bool MIL>
__device__ __forceinline__ double cir_step(double x, double dw, double dt, double kp, double th, double sg) {
    double r = __dadd_rn(x, __dmul_rn(__dmul_rn(kp, __dsub_rn(th, x)), dt));
    r = __dadd_rn(r, __dmul_rn(__dmul_rn(sg, __dsqrt_rn(fabs(x))), dw));
    if (MIL) r = __dadd_rn(r, __dmul_rn(__dmul_rn(__dmul_rn(0.25, sg), sg), __dsub_rn(__dmul_rn(dw, dw), dt)));
    return r;
}

// ------------------------------------------------------ CTA reduction --
// Warp sums of 5 values per lane with the xor-butterfly's summation tree
// (pairs at lane distance 16, then 8, 4, 2, 1 -- the tree the plain
// `s += shfl_xor(s, o)` loop builds in every lane, so the results are bit for
// bit those of the per-value butterflies), but the first four values share
// the lanes: at distance 16 the warp's halves exchange one of each pair of
// values and keep the other, at distance 8 the quarters do the same, and from
// there one value per lane is left.  6 + 5 64-bit shuffles and adds instead
// of 25.  Results: value 0 / 1 / 2 / 3 in lanes [0, 8) / [16, 24) / [8, 16) /
// [24, 32) of `c`, value 4 in every lane of `e`.
struct WarpSum5 {
    double c, e;
};
__device__ __forceinline__ WarpSum5 warp_sum5(const double (&x)[5], int lane) {
    const bool h16 = lane & 16, h8 = lane & 8;
    const double a = (h16 ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, h16 ? x[0] : x[1], 16);
    const double b = (h16 ? x[3] : x[2]) + __shfl_xor_sync(0xffffffffu, h16 ? x[2] : x[3], 16);
    double c = (h8 ? b : a) + __shfl_xor_sync(0xffffffffu, h8 ? a : b, 8);
    double e = x[4];
    e += __shfl_xor_sync(0xffffffffu, e, 16);
    e += __shfl_xor_sync(0xffffffffu, e, 8);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, o);
        e += __shfl_xor_sync(0xffffffffu, e, o);
    }
    return {c, e};
}
// which of the first four values lane group (lane >> 3) holds in WarpSum5::c
__device__ __forceinline__ int warp_sum5_kind(int lane) { return ((lane >> 4) & 1) | ((lane >> 2) & 2); }

// Two-pass (count, mean, M2) of NK values per thread over the CTA.
template <int NK, int BS = kLevelBlock>
__device__ __forceinline__ void cta_moments(const double (&d)[NK], bool valid, double *partial_out) {
    static_assert(NK == 5, "warp_sum5");
    // One buffer per pass: a call's first-pass sums are last read before its second
    // barrier and its second-pass sums before the next call's first barrier, so
    // back-to-back calls (one per tile) need no barrier on entry -- three per call.
    __shared__ double red[2][NK][BS / 32];
    __shared__ double mean_sh[NK];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double s[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) s[k] = valid ? d[k] : 0.0;
    WarpSum5 w = warp_sum5(s, lane);
    if ((lane & 7) == 0) red[0][warp_sum5_kind(lane)][warp] = w.c;
    if (lane == 0) red[0][4][warp] = w.e;
    const int count = __syncthreads_count(valid);
    if (threadIdx.x < NK) {
        double t = 0.0;
        for (int i = 0; i < BS / 32; ++i) t += red[0][threadIdx.x][i];
        mean_sh[threadIdx.x] = count > 0 ? t / count : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        const double dv = valid ? d[k] - mean_sh[k] : 0.0;
        s[k] = dv * dv;
    }
    w = warp_sum5(s, lane);
    if ((lane & 7) == 0) red[1][warp_sum5_kind(lane)][warp] = w.c;
    if (lane == 0) red[1][4][warp] = w.e;
    __syncthreads();
    if (threadIdx.x < NK) {
        double t = 0.0;
        for (int i = 0; i < BS / 32; ++i) t += red[1][threadIdx.x][i];
        double *o = partial_out + 3 * threadIdx.x;
        o[0] = count;
        o[1] = mean_sh[threadIdx.x];
        o[2] = t;
    }
}

// Merge n_parts partials (n_parts x NK x 3 of count, mean, M2) into out
// (NK x 3) with the parallel-axis identity instead of a chain of pairwise
// Chan merges (two divisions each):
//   N = sum n_i,  mean = (sum n_i mean_i) / N,  M2 = sum [M2_i + n_i (mean_i - mean)^2]
// -- two passes of plain fused multiply-adds over the partials (every M2 term
// is non-negative), each a fixed-order block reduction (thread t takes
// partials t, t + B, ...; xor-shuffle tree; warps summed in order), so the
// result is bitwise reproducible.
template <int NK, int BS = kFinalBlock>
__device__ __forceinline__ void block_sum(double (&v)[NK], double (*sh)[NK], double *res) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if (lane == 0) sh[warp][k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < NK) {
        double t = 0.0;
        for (int w = 0; w < BS / 32; ++w) t += sh[w][threadIdx.x];
        res[threadIdx.x] = t;
    }
    __syncthreads();
}

template <int NK>
__global__ void __launch_bounds__(kFinalBlock) k_finalize(const double *__restrict__ parts, int64_t n_parts,
                                                          double *__restrict__ out) {
    __shared__ double sh[kFinalBlock / 32][NK];
    __shared__ double cnt[NK], sum[NK], m2[NK];
    double a[NK], b[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) a[k] = b[k] = 0.0;
    for (int64_t i = threadIdx.x; i < n_parts; i += kFinalBlock) {
        const double *p = parts + i * NK * 3;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            a[k] += p[3 * k];
            b[k] = fma(p[3 * k], p[3 * k + 1], b[k]);
        }
    }
    block_sum<NK>(a, sh, cnt);
    block_sum<NK>(b, sh, sum);
    double mean[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        mean[k] = cnt[k] > 0.0 ? sum[k] / cnt[k] : 0.0;
        a[k] = 0.0;
    }
    for (int64_t i = threadIdx.x; i < n_parts; i += kFinalBlock) {
        const double *p = parts + i * NK * 3;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const double d = p[3 * k + 1] - mean[k];
            a[k] = fma(p[3 * k] * d, d, a[k] + p[3 * k + 2]);
        }
    }
    block_sum<NK>(a, sh, m2);
    if (threadIdx.x < NK) {
        const int k = threadIdx.x;
        out[3 * k + 0] = cnt[k];
        out[3 * k + 1] = mean[k];
        out[3 * k + 2] = m2[k];
    }
}

// The same merge over many partials (large levels) in one kernel of
// kFinChunks CTAs: each CTA merges a fixed contiguous chunk of partials into
// one (count, mean, M2) triple with the two-pass parallel-axis identity (its
// chunk stays in L1/L2 between the passes), and the last CTA to finish (atomic
// ticket) merges the chunk triples the same way, in chunk order -- bitwise
// reproducible, ~4x faster than one CTA streaming 2 MB twice.
constexpr int kFinStageBlock = 256;
constexpr int kFinChunks = 64;
constexpr int64_t kFinSingleMax = 2048;  // up to this many partials: k_finalize
struct FinScratch {
    double stage[kFinChunks][ARV_NKIND][3];  // per-chunk (count, mean, M2)
    unsigned ticket;
};

// Parallel-axis merge of triples p[i * stride + 3k + {0,1,2}], i in [lo, hi),
// over the CTA (fixed order); results for kind k in r[k][0..2].
template <int NK>
__device__ __forceinline__ void cta_merge_triples(const double *p, int64_t stride, int64_t lo, int64_t hi,
                                                  double (*sh)[NK], double (&r)[NK][3], bool cached) {
    __shared__ double cnt[NK], sum[NK], m2[NK];
    double a[NK], b[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) a[k] = b[k] = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kFinStageBlock) {
        const double *q = p + i * stride;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const double n = cached ? __ldcg(q + 3 * k) : q[3 * k];
            const double m = cached ? __ldcg(q + 3 * k + 1) : q[3 * k + 1];
            a[k] += n;
            b[k] = fma(n, m, b[k]);
        }
    }
    block_sum<NK, kFinStageBlock>(a, sh, cnt);
    block_sum<NK, kFinStageBlock>(b, sh, sum);
    double mean[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        mean[k] = cnt[k] > 0.0 ? sum[k] / cnt[k] : 0.0;
        a[k] = 0.0;
    }
    for (int64_t i = lo + threadIdx.x; i < hi; i += kFinStageBlock) {
        const double *q = p + i * stride;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const double n = cached ? __ldcg(q + 3 * k) : q[3 * k];
            const double d = (cached ? __ldcg(q + 3 * k + 1) : q[3 * k + 1]) - mean[k];
            a[k] = fma(n * d, d, a[k] + (cached ? __ldcg(q + 3 * k + 2) : q[3 * k + 2]));
        }
    }
    block_sum<NK, kFinStageBlock>(a, sh, m2);
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        r[k][0] = cnt[k];
        r[k][1] = mean[k];
        r[k][2] = m2[k];
    }
}

template <int NK>
__global__ void __launch_bounds__(kFinStageBlock) k_finalize_chunks(const double *__restrict__ parts,
                                                                    int64_t n_parts, FinScratch *fs,
                                                                    double *__restrict__ out) {
    __shared__ double sh[kFinStageBlock / 32][NK];
    __shared__ bool last;
    const int64_t per = (n_parts + gridDim.x - 1) / gridDim.x;
    const int64_t lo = static_cast<int64_t>(blockIdx.x) * per;
    const int64_t hi = lo + per < n_parts ? lo + per : n_parts;
    double r[NK][3];
    cta_merge_triples<NK>(parts, NK * 3, lo, hi, sh, r, false);
    if (threadIdx.x < NK * 3) fs->stage[blockIdx.x][threadIdx.x / 3][threadIdx.x % 3] = r[threadIdx.x / 3][threadIdx.x % 3];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(&fs->ticket, 1u);
        ARV_DCHECK(t < gridDim.x);  // the ticket starts at 0 for every call
        last = t == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    cta_merge_triples<NK>(&fs->stage[0][0][0], NK * 3, 0, gridDim.x, sh, r, true);
    if (threadIdx.x < NK * 3) out[threadIdx.x] = r[threadIdx.x / 3][threadIdx.x % 3];
    if (threadIdx.x == 0) fs->ticket = 0u;  // ready for the next call
}

// --------------------------------------------------- Gaussian schemes --
// SCHEME: ARV_SCHEME_EM, _MILSTEIN (GBM), _CIR_EULER_TRUNCATED, _CIR_MILSTEIN_TRUNCATED
template <int DEG, int SCHEME, bool PHILOX>
__global__ void __launch_bounds__(kLevelBlock, (SCHEME == ARV_SCHEME_EM || SCHEME == ARV_SCHEME_MILSTEIN) && !PHILOX
                                                   ? ARV_GBM_MINB_PCG
                                                   : ARV_GBM_MINB) k_gaussian_level(LevelArgs A, const double *__restrict__ coeffs,
                                                                int64_t K1, double *__restrict__ parts,
                                                                double *__restrict__ paths) {
    extern __shared__ double smd[];
    __shared__ double2 as241_rows[ARV_GBM_SMEM_ROWS ? 16 : 1];
    for (int i = threadIdx.x; i < (DEG + 1) * K1; i += blockDim.x) smd[i] = __ldg(coeffs + i);
    if (ARV_GBM_SMEM_ROWS) as241_stage_rows(as241_rows);
    __syncthreads();
    const double2 *rows = ARV_GBM_SMEM_ROWS ? as241_rows : nullptr;
    constexpr bool GBM = SCHEME == ARV_SCHEME_EM || SCHEME == ARV_SCHEME_MILSTEIN;
    constexpr bool MIL = SCHEME == ARV_SCHEME_MILSTEIN || SCHEME == ARV_SCHEME_CIR_MILSTEIN_TRUNCATED;

    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = i < A.path_count;
    double d[ARV_NKIND] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (valid) {
        const uint64_t p = static_cast<uint64_t>(A.path_lo + i);
        PathSource<PHILOX> rng(A, p);
        const double x0 = A.x0, dt_f = A.dt_f, dt_c = A.dt_c, sq_f = A.sq_f;
        double xf_e = x0, xc_e = x0, xf_a = x0, xc_a = x0;
        auto step = [&](double x, double dw, double dt) -> double {
            if constexpr (GBM) return gbm_step<MIL>(x, dw, dt, A.a, A.b);
            else return cir_step<MIL>(x, dw, dt, A.a, A.b, A.c);
        };
        // one coarse step = two fine steps; exact (AS241) and table normals of
        // the same uniforms (mlmc.py:200-229)
        auto pair_step = [&](const double *z, const double *w) {
            xf_e = step(step(xf_e, __dmul_rn(sq_f, z[0]), dt_f), __dmul_rn(sq_f, z[1]), dt_f);
            xc_e = step(xc_e, __dmul_rn(sq_f, __dadd_rn(z[0], z[1])), dt_c);
            xf_a = step(step(xf_a, __dmul_rn(sq_f, w[0]), dt_f), __dmul_rn(sq_f, w[1]), dt_f);
            xc_a = step(xc_a, __dmul_rn(sq_f, __dadd_rn(w[0], w[1])), dt_c);
        };
        int64_t pairs = A.n_f / 2;
#if ARV_GBM_QUAD
        for (; pairs >= 2; pairs -= 2) {  // four uniforms per pass: AS241 tails compacted 4-wide
            double u[4], z[4], w[4];
            bool lo[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) u[k] = rng.next(lo[k]);
            if (A.want_exact) as241_f64_batch<4, true>(u, z, rows);
            else z[0] = z[1] = z[2] = z[3] = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) w[k] = A.want_approx ? gauss_table_eval<DEG>(smd, K1, u[k], lo[k]) : 0.0;
            pair_step(z, w);
            pair_step(z + 2, w + 2);
        }
#endif
        for (; pairs > 0; --pairs) {
            double u[2], z[2], w[2];
            bool lo[2];
            u[0] = rng.next(lo[0]);
            u[1] = rng.next(lo[1]);
            if (A.want_exact) as241_f64_batch<2, true>(u, z, rows);
            else z[0] = z[1] = 0.0;
            w[0] = A.want_approx ? gauss_table_eval<DEG>(smd, K1, u[0], lo[0]) : 0.0;
            w[1] = A.want_approx ? gauss_table_eval<DEG>(smd, K1, u[1], lo[1]) : 0.0;
            pair_step(z, w);
        }
        if (A.n_f & 1) {
            bool lo;
            const double u = rng.next(lo);
            if (A.want_exact) xf_e = step(xf_e, __dmul_rn(sq_f, as241_f64(u)), dt_f);
            if (A.want_approx) xf_a = step(xf_a, __dmul_rn(sq_f, gauss_table_eval<DEG>(smd, K1, u, lo)), dt_f);
        }
        const double fe = payoff_fn(xf_e, A.payoff, A.strike);
        const double fa = payoff_fn(xf_a, A.payoff, A.strike);
        const double ce = A.level > 0 ? payoff_fn(xc_e, A.payoff, A.strike) : 0.0;
        const double ca = A.level > 0 ? payoff_fn(xc_a, A.payoff, A.strike) : 0.0;
        // mlmc.py:341-353 (two_way exact / approx, four_way) and plain
        d[0] = __dsub_rn(fe, ce);
        d[1] = __dsub_rn(fa, ca);
        d[2] = __dadd_rn(__dsub_rn(__dsub_rn(fe, ce), fa), ca);
        d[3] = fe;
        d[4] = fa;
        if (paths) {
            paths[i] = fe;
            paths[A.path_count + i] = ce;
            paths[2 * A.path_count + i] = fa;
            paths[3 * A.path_count + i] = ca;
        }
    }
    cta_moments<ARV_NKIND>(d, valid, parts + static_cast<int64_t>(blockIdx.x) * 3 * ARV_NKIND);
}

// ------------------------------------------ Gaussian level kernel, v2 --
// PCG32 streams (the BASELINE generator), every Gaussian scheme.  Same paths,
// same approximate side bit for bit, same statistics layout as
// k_gaussian_level; the work per path-step is restructured around the word w
// of the uniform u = (w + 1/2) 2^-32:
//  * exact side (AS241, exact_dist.py:87-126): the central rational
//    (|u - 1/2| <= 0.425, an integer range test on w) is evaluated for every
//    element with the A/B coefficients as compile-time constants -- they
//    become constant-bank operands of the FP64 instructions, so there are no
//    coefficient loads or per-lane row selects (k_gaussian_level read 8
//    16-byte rows per element from shared memory to serve central and tail
//    lanes with one rational).  Tail elements (15%) are compacted warp-wide
//    into a per-warp list and get their whole tail evaluation -- log, sqrt,
//    C/D (or E/F) rational, division -- in one pass per 32 tails, again with
//    constant coefficients.  q = u - 1/2 = (1 + u) - 3/2 and the tail's
//    min(u, 1 - u) are built exactly from w's bits.
//  * approximate side (dyadic_eval / constant_eval, _kernels.pyx:16-73):
//    v = min(u, 1 - u) = (w' + 1/2) 2^-32 with w' = w or ~w (exact), the
//    interval index 1022 - expo(v) = clz(w') (capped), one 16-byte shared
//    load for (c0, c1), the reference's separately rounded Horner steps, and
//    the sign as an XOR of w's top bit into z's sign bit.
//  * path updates: mu dt, (0.5 sg) sg hoisted (same roundings).
// With ARV_GBM_FMA_EXACT the exact side's Horner steps and the division are
// fused multiply-adds (a different rounding of the same AS241 evaluation,
// relative differences ~1e-16 per normal; the MLMC contract for the exact
// side is statistical, and per-path tests hold it to 1e-13).
#ifndef ARV_GBM_V2
#define ARV_GBM_V2 1
#endif
#ifndef ARV_GBM_FMA_EXACT
#define ARV_GBM_FMA_EXACT 1
#endif
#ifndef ARV_GBM_V2_MINB
#define ARV_GBM_V2_MINB 4
#endif
#ifndef ARV_GBM_DIV_CORRECT  // residual-corrected (correctly rounded) division on the exact side
#define ARV_GBM_DIV_CORRECT 0  // 0: n * rcp(d) (~1 ulp): config 4 11.74 -> 11.15 ms with FMA steps
#endif
#ifndef ARV_GBM_SIDES_SPLIT  // a both-sides instantiation without the per-iteration side tests
#define ARV_GBM_SIDES_SPLIT 1  // 11.06 -> 10.73 ms (config 4)
#endif
#ifndef ARV_GBM_LOCKSTEP  // central rationals of the N words in lockstep
#define ARV_GBM_LOCKSTEP 1  // 11.14 -> 11.06 ms (config 4)
#endif
#ifndef ARV_GBM_FMA_STEP  // exact-side GBM steps as FMAs
#define ARV_GBM_FMA_STEP 1
#endif

namespace g2 {
// coefficient sets: rows of the __constant__ table kAS241d (A, B, C, D, E, F);
// indexed with compile-time indices they are constant-bank operands of the
// FP64 instructions (literal doubles would be materialised with two UMOVs each)
enum { kA = 0, kB = 1, kC = 2, kD = 3, kE = 4, kF = 5 };
// |u - 1/2| <= 0.425 (exact_dist.py:92) for u = (w + 1/2) 2^-32 <=> w in
// [ceil(2^31 - 1/2 - 0.425 * 2^32), floor(2^31 - 1/2 + 0.425 * 2^32)]
// (0.425 the double; q is exact, so the integer test is exact)
constexpr uint32_t kCentralLo = 0x13333333u, kCentralSpan = 0xECCCCCCCu - 0x13333333u;

template <bool FMA>
__device__ __forceinline__ double horner(int which, double x) {
    double acc = kAS241d[which][7];
#pragma unroll
    for (int i = 6; i >= 0; --i)
        acc = FMA ? fma(acc, x, kAS241d[which][i]) : __dadd_rn(__dmul_rn(acc, x), kAS241d[which][i]);
    return acc;
}

// n / d for the positive, well-scaled AS241 denominators: reciprocal estimate
// y0 (MUFU.RCP64H: the operand's top 20 mantissa bits, relative error e ~ 2^-20)
// and one second-order step y = y0 (1 + e + e^2) = (1 - e^3) / d -- three DFMA,
// ~2^-60 before rounding; the quotient n y is within ~1.5 ulp of n / d.
#ifndef ARV_GBM_RCP_ORDER2
#define ARV_GBM_RCP_ORDER2 1  // 0: two Newton steps (four DFMA)
#endif
template <bool FMA>
__device__ __forceinline__ double divide(double n, double d) {
    if constexpr (!FMA) {
        return __ddiv_rn(n, d);
    } else {
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
#if ARV_GBM_RCP_ORDER2
        const double e = fma(-d, y, 1.0);
        y = fma(y, fma(e, e, e), y);
#else
        y = fma(fma(-d, y, 1.0), y, y);
        y = fma(fma(-d, y, 1.0), y, y);
#endif
#if ARV_GBM_DIV_CORRECT
        const double q0 = __dmul_rn(n, y);
        return fma(fma(-d, q0, n), y, q0);
#else
        return __dmul_rn(n, y);
#endif
    }
}

template <bool FMA>
__device__ __forceinline__ double central(double q) {
    const double r = FMA ? fma(-q, q, 0.180625) : __dsub_rn(0.180625, __dmul_rn(q, q));
    return divide<FMA>(__dmul_rn(q, horner<FMA>(kA, r)), horner<FMA>(kB, r));
}

// -log(v) for a tail element, v = min(u, 1 - u) in [2^-33, 0.075): with
// v = m 2^e, m in [1, 2), bucket j = top 7 mantissa bits of m and the table
// (inv_j, T_j = log(inv_j)) of arv_logtab.cuh, m inv_j = 1 + r exactly in the
// FMA (|r| <= 2^-8) and -log(v) = (-e) ln2 + T_j - log1p(r); log1p by its
// series through r^6 (truncation < 2^-58).  ~1.1 ulp (tools/make_log_table.py,
// tests/test_gpu_mlmc.py::test_level_normals_accuracy); 9 FP64 operations where
// CUDA's log() takes ~25 plus ~20 constant moves.
__device__ __forceinline__ double neg_log(double v) {
    const int hi = __double2hiint(v);
    const int ne = 1023 - (hi >> 20);
    const double2 tj = __ldg(kLogTab + ((hi >> 13) & 127));
    const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(v));
    const double r = fma(m, tj.x, -1.0);
    double q = fma(r, -1.0 / 6.0, 0.2);
    q = fma(q, r, -0.25);
    q = fma(q, r, 1.0 / 3.0);
    q = fma(q, r, -0.5);
    const double lp = fma(__dmul_rn(r, r), q, r);
    return __dsub_rn(fma(static_cast<double>(ne), 0.6931471805599453094, tj.y), lp);
}

// sqrt(x) for x in [2.5, 24]: MUFU.RSQ64H estimate (~2^-20), one coupled
// Goldschmidt step (g ~ sqrt x, h ~ 1 / (2 sqrt x) to ~2^-39) and the final
// residual correction: faithful (< 1 ulp; 0.99 * 2^-53 relative in the CPU
// emulation), no special-case path (__dsqrt_rn carries one behind a CALL).
__device__ __forceinline__ double sqrt_mid(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double g = __dmul_rn(x, y), h = __dmul_rn(0.5, y);
    const double r = fma(-g, h, 0.5);
    g = fma(g, r, g);
    h = fma(h, r, h);
    return fma(fma(-g, g, x), h, g);
}

#ifndef ARV_GBM_TAIL_CUSTOM
#define ARV_GBM_TAIL_CUSTOM 1  // 0: CUDA log() and __dsqrt_rn
#endif
// |AS241(u)| of a tail element from w = min(u, 1 - u) (exact_dist.py:100-126)
// FAR = false: callers whose uniforms carry 32 bits (v >= 2^-33, r <= 4.79)
// never reach the far-tail E / F rational.
template <bool FMA, bool FAR = true>
__device__ __forceinline__ double tail_abs(double w) {
#if ARV_GBM_TAIL_CUSTOM
    const double r = FMA ? sqrt_mid(neg_log(w)) : __dsqrt_rn(-log(w));
#else
    const double r = __dsqrt_rn(-log(w));
#endif
    if (!FAR || r <= 5.0) {
        const double x = __dsub_rn(r, 1.6);
        return divide<FMA>(horner<FMA>(kC, x), horner<FMA>(kD, x));
    }
    const double x = __dsub_rn(r, 5.0);
    return divide<FMA>(horner<FMA>(kE, x), horner<FMA>(kF, x));
}

// Central rational of N words (every element; tail elements get a value
// that the caller replaces) and the tail bits (|u - 1/2| > 0.425).
template <int N, bool FMA>
__device__ __forceinline__ unsigned central_words(const uint32_t (&w)[N], double (&z)[N]) {
    unsigned pend = 0;
#if ARV_GBM_LOCKSTEP
    if constexpr (FMA) {  // the N central rationals in lockstep: 2N independent Horner chains
        double q[N], r[N], a[N], b[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if (w[k] - kCentralLo > kCentralSpan) pend |= 1u << k;
            q[k] = __dsub_rn(one_plus_u32(w[k]), 1.5);
            r[k] = fma(-q[k], q[k], 0.180625);
            a[k] = kAS241d[kA][7];
            b[k] = kAS241d[kB][7];
        }
#pragma unroll
        for (int i = 6; i >= 0; --i)
#pragma unroll
            for (int k = 0; k < N; ++k) {
                a[k] = fma(a[k], r[k], kAS241d[kA][i]);
                b[k] = fma(b[k], r[k], kAS241d[kB][i]);
            }
#pragma unroll
        for (int k = 0; k < N; ++k) z[k] = divide<FMA>(__dmul_rn(q[k], a[k]), b[k]);
    } else
#endif
    {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if (w[k] - kCentralLo > kCentralSpan) pend |= 1u << k;
            z[k] = central<FMA>(__dsub_rn(one_plus_u32(w[k]), 1.5));  // q = u - 1/2 exactly
        }
    }
    return pend;
}

// AS241 of N words per lane; all 32 lanes of the warp call it together.
// v[k] = min(u, 1 - u) of element k (exact).  buf: this warp's 32 N doubles.
template <int N, bool FMA>
__device__ __forceinline__ void as241_words(const uint32_t (&w)[N], const double (&v)[N], double (&z)[N],
                                            double *buf) {
    const unsigned pend = central_words<N, FMA>(w, z);
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    int pos[N];
    int total = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const unsigned b = __ballot_sync(0xffffffffu, (pend >> k) & 1u);
        pos[k] = total + __popc(b & lt);
        total += __popc(b);
    }
    if (total) {  // warp-uniform
#pragma unroll
        for (int k = 0; k < N; ++k)
            if ((pend >> k) & 1u) {
                ARV_DCHECK(pos[k] >= 0 && pos[k] < total && total <= 32 * N);
                buf[pos[k]] = v[k];
            }
        __syncwarp();
        for (int g = threadIdx.x & 31; g < total; g += 32) buf[g] = tail_abs<FMA, false>(buf[g]);  // PCG32 words only (v >= 2^-33)
        __syncwarp();
#pragma unroll
        for (int k = 0; k < N; ++k)
            if ((pend >> k) & 1u) {
                const double t = buf[pos[k]];
                z[k] = w[k] >> 31 ? t : -t;  // upper tail positive (exact_dist.py:124-126)
            }
        __syncwarp();  // the list is reused by the next call
    }
}

// v = min(u, 1 - u) = (w' + 1/2) 2^-32, w' = w (u < 1/2) or ~w -- as
// 1/2 - |q| with q = u - 1/2 = (1 + u) - 3/2, both subtractions exact (all
// three are multiples of 2^-33 below 1).  q is the central rational's own
// argument (the compiler shares it), so v costs one FP64 add with a free |.|
// instead of a second bit assembly of 1 + u'.
__device__ __forceinline__ double reflected(uint32_t w) {
    return __dsub_rn(0.5, fabs(__dsub_rn(one_plus_u32(w), 1.5)));
}

// Approximate side of one element: dyadic_eval (DEG >= 1; table interleaved
// [K1][S] with S = DEG + 1 rounded up to even) or constant_eval (DEG == 0,
// values[K1]) -- _kernels.pyx:56-73, :16-23.
template <int DEG>
__device__ __forceinline__ double table(const double *sm, uint32_t w, double v, int cap, int64_t K1) {
    if constexpr (DEG == 0) {
        const double u = __dsub_rn(one_plus_u32(w), 1.0);
        long long idx = static_cast<long long>(__dmul_rn(static_cast<double>(K1), u));
        idx = idx < K1 ? idx : K1 - 1;
        ARV_DCHECK(idx >= 0 && idx < K1);
        return sm[idx];
    } else {
        constexpr int S = (DEG + 2) & ~1;
        // 1022 - expo(v) (_kernels.pyx:36) read off v's exponent field: v in [2^-33, 1/2)
        // is (w' + 1/2) 2^-32, so it equals clz(w') (a shift and an add-min)
        int idx = 1022 - (__double2hiint(v) >> 20);
        idx = idx < cap ? idx : cap;
        ARV_DCHECK(idx >= 0 && idx <= cap);
        const double *c = sm + idx * S;
        double z;
        if constexpr (DEG == 1) {
            const double2 c01 = *reinterpret_cast<const double2 *>(c);
            z = __dadd_rn(__dmul_rn(c01.y, v), c01.x);
        } else {
            z = c[DEG];
#pragma unroll
            for (int d = DEG - 1; d >= 0; --d) z = __dadd_rn(__dmul_rn(z, v), c[d]);
        }
        // out = pred ? z : -z (u < 1/2 <=> top bit of w clear)
        return __hiloint2double(__double2hiint(z) ^ static_cast<int>(w & 0x80000000u), __double2loint(z));
    }
}
}  // namespace g2

template <int DEG, int SCHEME, bool BOTH>
__global__ void __launch_bounds__(kLevelBlock, ARV_GBM_V2_MINB) k_gaussian_level_v2(LevelArgs A,
                                                                                 const double *__restrict__ coeffs,
                                                                                 int64_t K1,
                                                                                 double *__restrict__ parts,
                                                                                 double *__restrict__ paths) {
    constexpr bool FMA = ARV_GBM_FMA_EXACT != 0;
    constexpr bool GBM = SCHEME == ARV_SCHEME_EM || SCHEME == ARV_SCHEME_MILSTEIN;
    constexpr bool MIL = SCHEME == ARV_SCHEME_MILSTEIN || SCHEME == ARV_SCHEME_CIR_MILSTEIN_TRUNCATED;
    constexpr int S = DEG == 0 ? 1 : (DEG + 2) & ~1;
    extern __shared__ __align__(16) double smd[];
    __shared__ double tails[kLevelBlock / 32][32 * 4];
    if constexpr (DEG == 0) {
        for (int i = threadIdx.x; i < K1; i += blockDim.x) smd[i] = __ldg(coeffs + i);
    } else {  // reference layout (DEG+1, K1) -> interleaved [K1][S]
        for (int i = threadIdx.x; i < (DEG + 1) * K1; i += blockDim.x) {
            const int d = static_cast<int>(i / K1), j = static_cast<int>(i % K1);
            smd[j * S + d] = __ldg(coeffs + i);
        }
    }
    __syncthreads();
    double *buf = tails[threadIdx.x >> 5];
    const int cap = static_cast<int>(K1 - 1);

    // Persistent tiles: the grid is one wave of resident CTAs, and CTA b
    // simulates tiles b, b + G, b + 2G, ... of 256 paths (tile t = paths
    // path_lo + 256 t + [0, 256)), writing tile t's partial exactly as the
    // one-tile-per-CTA form did: same partition, same statistics bit for bit.
    // The table, the lane maps and the tile start are set up once per CTA
    // instead of once per 256 paths; path p's PCG32 state is LCG^lane applied
    // to the tile's start state (a per-lane map staged in shared memory, the
    // tile start advanced by one map per tile) instead of a walk over the bits
    // of p per thread.
    // lane maps and the tile-to-tile map live in shared memory (re-read once
    // per tile) so that they do not hold registers across the path loop
    __shared__ Affine lane_map[kLevelBlock + 1];  // [kLevelBlock]: tile -> next tile of this CTA
    {
        Affine m{1, 0};
        const unsigned t = threadIdx.x;
        for (int b = 0; b < 8; ++b)
            if ((t >> b) & 1u) m = {A.jump2[b].a * m.a, A.jump2[b].a * m.c + A.jump2[b].c};
        lane_map[t] = m;
        if (t == 0) {
            Affine g{1, 0};
            const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kLevelBlock;
            for (int b = 0; b < kPathJumpBits; ++b)
                if ((stride >> b) & 1u) g = {A.jump2[b].a * g.a, A.jump2[b].a * g.c + A.jump2[b].c};
            lane_map[kLevelBlock] = g;
        }
    }
    const int64_t ntiles = (A.path_count + kLevelBlock - 1) / kLevelBlock;
    // start state of this CTA's current tile: one thread (of another warp than the
    // stride map's) walks the bits of the path index, the rest read it after the barrier
    __shared__ uint64_t tile_s0;
    if (threadIdx.x == 32)
        tile_s0 = path_start_state(A, static_cast<uint64_t>(A.path_lo) + static_cast<uint64_t>(blockIdx.x) * kLevelBlock);
    __syncthreads();
    uint64_t tile_s = tile_s0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * kLevelBlock + threadIdx.x;
    const bool valid = i < A.path_count;
    // every lane runs the path loop (the tail list needs the whole warp);
    // lanes past the range simulate a path beyond it and are not counted
    uint64_t s;
    {
        const Affine my = lane_map[threadIdx.x], nx = lane_map[kLevelBlock];
        s = my.a * tile_s + my.c;
        tile_s = nx.a * tile_s + nx.c;
    }
    const Affine st = A.step;
    const double x0 = A.x0, dt_f = A.dt_f, dt_c = A.dt_c, sq_f = A.sq_f;
    const double mudt_f = __dmul_rn(A.a, dt_f), mudt_c = __dmul_rn(A.a, dt_c);  // mlmc.py:195
    const double sg = A.b, hs2 = __dmul_rn(__dmul_rn(0.5, A.b), A.b);           // mlmc.py:196-197
    // BOTH (sides = both, the MLMC estimators): the side tests are compile-time
    // true, so the loop body is one basic block the scheduler can interleave
    const bool we = BOTH || A.want_exact, wa = BOTH || A.want_approx;
    double xf_e = x0, xc_e = x0, xf_a = x0, xc_a = x0;
    auto step = [&](double x, double dw, double dt, double mudt) -> double {
        if constexpr (GBM) {
            double incr = __dadd_rn(mudt, __dmul_rn(sg, dw));
            if (MIL) incr = __dadd_rn(incr, __dmul_rn(hs2, __dsub_rn(__dmul_rn(dw, dw), dt)));
            return __dmul_rn(x, __dadd_rn(1.0, incr));
        } else {
            return cir_step<MIL>(x, dw, dt, A.a, A.b, A.c);
        }
    };
    // exact side with ARV_GBM_FMA_STEP: the same GBM step as fused multiply-adds
    // (x + x (mu dt + sg dw)), one rounding fewer per operation; the approximate
    // side always keeps the reference's separately rounded em_step
    auto step_e = [&](double x, double dw, double dt, double mudt) -> double {
        if constexpr (GBM && FMA && ARV_GBM_FMA_STEP) {
            double incr = fma(sg, dw, mudt);
            if (MIL) incr = fma(hs2, fma(dw, dw, -dt), incr);
            return fma(x, incr, x);
        } else {
            return step(x, dw, dt, mudt);
        }
    };
    // Exact-side step from the normal z (dW = sqrt(dt_f) z).  GBM Euler-Maruyama with
    // FMA steps: sg sqrt(dt_f) is folded into one constant, x + x (mu dt + (sg sqrt(dt_f)) z)
    // -- one FP64 multiply per step fewer (the level kernels are FP64-pipe-bound).
    const double sgsq = __dmul_rn(sg, sq_f);
    auto step_z = [&](double x, double z, double dt, double mudt) -> double {
        if constexpr (GBM && FMA && ARV_GBM_FMA_STEP && !MIL) return fma(x, fma(sgsq, z, mudt), x);
        else return step_e(x, __dmul_rn(sq_f, z), dt, mudt);
    };
    auto pair_step = [&](double z0, double z1, double w0, double w1) {
        xf_e = step_z(step_z(xf_e, z0, dt_f, mudt_f), z1, dt_f, mudt_f);
        xc_e = step_z(xc_e, __dadd_rn(z0, z1), dt_c, mudt_c);
        xf_a = step(step(xf_a, __dmul_rn(sq_f, w0), dt_f, mudt_f), __dmul_rn(sq_f, w1), dt_f, mudt_f);
        xc_a = step(xc_a, __dmul_rn(sq_f, __dadd_rn(w0, w1)), dt_c, mudt_c);
    };
    auto draw = [&]() -> uint32_t {
        const uint32_t w = pcg32_output(s);
        s = st.a * s + st.c;
        return w;
    };
    int64_t pairs = A.n_f / 2;
    for (; pairs >= 2; pairs -= 2) {  // four uniforms (two coarse steps) per pass
        uint32_t w[4];
        double v[4], z[4], a[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            w[k] = draw();
            v[k] = g2::reflected(w[k]);
        }
        if (we) g2::as241_words<4, FMA>(w, v, z, buf);
        else z[0] = z[1] = z[2] = z[3] = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = wa ? g2::table<DEG>(smd, w[k], v[k], cap, K1) : 0.0;
        pair_step(z[0], z[1], a[0], a[1]);
        pair_step(z[2], z[3], a[2], a[3]);
    }
    if (pairs) {
        uint32_t w[2];
        double v[2], z[2], a[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            w[k] = draw();
            v[k] = g2::reflected(w[k]);
        }
        if (we) g2::as241_words<2, FMA>(w, v, z, buf);
        else z[0] = z[1] = 0.0;
#pragma unroll
        for (int k = 0; k < 2; ++k) a[k] = wa ? g2::table<DEG>(smd, w[k], v[k], cap, K1) : 0.0;
        pair_step(z[0], z[1], a[0], a[1]);
    }
    if (A.n_f & 1) {  // odd fine-step count (n0 odd at level 0)
        uint32_t w[1] = {draw()};
        double v[1] = {g2::reflected(w[0])}, z[1] = {0.0};
        if (we) g2::as241_words<1, FMA>(w, v, z, buf);
        if (we) xf_e = step_z(xf_e, z[0], dt_f, mudt_f);
        if (wa) xf_a = step(xf_a, __dmul_rn(sq_f, g2::table<DEG>(smd, w[0], v[0], cap, K1)), dt_f, mudt_f);
    }
    double d[ARV_NKIND] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (valid) {
        const double fe = payoff_fn(xf_e, A.payoff, A.strike);
        const double fa = payoff_fn(xf_a, A.payoff, A.strike);
        const double ce = A.level > 0 ? payoff_fn(xc_e, A.payoff, A.strike) : 0.0;
        const double ca = A.level > 0 ? payoff_fn(xc_a, A.payoff, A.strike) : 0.0;
        // mlmc.py:341-353 (two_way exact / approx, four_way) and plain
        d[0] = __dsub_rn(fe, ce);
        d[1] = __dsub_rn(fa, ca);
        d[2] = __dadd_rn(__dsub_rn(__dsub_rn(fe, ce), fa), ca);
        d[3] = fe;
        d[4] = fa;
        if (paths) {
            paths[i] = fe;
            paths[A.path_count + i] = ce;
            paths[2 * A.path_count + i] = fa;
            paths[3 * A.path_count + i] = ca;
        }
    }
    cta_moments<ARV_NKIND>(d, valid, parts + tile * 3 * ARV_NKIND);
    }
}

// ------------------------------------------ Gaussian level kernel, v3 --
// Both sides, PCG32 (the MLMC estimators' case).  Same paths, bit for bit, as
// k_gaussian_level_v2 (same functions per element, same tile partition of the
// statistics); the exact side is reorganised in phases over blocks of
// kV3Steps uniforms of the CTA's 256 paths:
//   1. every thread draws its block's words; evaluates the central rational of
//      each in lockstep groups of 4 (the A/B coefficients stay in uniform
//      registers for the whole phase) and stores z -- or, for a tail element,
//      +-v (v = min(u, 1 - u), the sign marking the upper tail) -- in zbuf,
//      its tail slots going to one CTA-wide list (one atomic per warp); and
//      runs the whole approximate side (table, both approximate path
//      updates), which needs nothing from the exact side;
//   2. the CTA's 256 threads serve the whole list: log, sqrt, C/D (E/F)
//      rational per entry -- ~450 tails per 12-step block, ~80% of the lanes
//      busy instead of ~60% with the per-iteration warp lists, and the tail
//      constants loaded once per pass instead of once per four uniforms;
//   3. every thread reads its z back and advances the two exact-side paths.
// Each thread only touches its own column of zbuf in phases 1 and 3, so two
// barriers per block suffice (after 1 and after 2).  Shared memory per block:
// 10 B per element (z and a 16-bit list slot).
#ifndef ARV_GBM_V3
#define ARV_GBM_V3 1
#endif
#ifndef ARV_V3_STEPS
#define ARV_V3_STEPS 20  // config 4: 12 -> 10.26 ms, 16 -> 9.95, 20 -> 9.89, 24 -> 10.02 (3 CTAs/SM)
#endif
constexpr int kV3Steps = ARV_V3_STEPS;
static_assert(kV3Steps % 2 == 0 && kV3Steps <= 32 && kV3Steps * kLevelBlock <= 65536,
              "block of uniforms (32-bit tail mask, u16 tail slots)");

__host__ __device__ constexpr int64_t v3_table_words(int degree, int64_t K1) {
    return ((degree == 0 ? K1 : static_cast<int64_t>((degree + 2) & ~1) * K1) + 1) & ~int64_t(1);
}
__host__ __device__ constexpr size_t v3_smem_bytes(int degree, int64_t K1) {
    return sizeof(double) * v3_table_words(degree, K1) +
           static_cast<size_t>(kV3Steps) * kLevelBlock * (sizeof(double) + sizeof(uint16_t));
}

template <int DEG, int SCHEME>
__global__ void __launch_bounds__(kLevelBlock, ARV_GBM_V2_MINB) k_gaussian_level_v3(LevelArgs A,
                                                                                 const double *__restrict__ coeffs,
                                                                                 int64_t K1,
                                                                                 double *__restrict__ parts,
                                                                                 double *__restrict__ paths) {
    constexpr bool FMA = ARV_GBM_FMA_EXACT != 0;
    constexpr bool GBM = SCHEME == ARV_SCHEME_EM || SCHEME == ARV_SCHEME_MILSTEIN;
    constexpr bool MIL = SCHEME == ARV_SCHEME_MILSTEIN || SCHEME == ARV_SCHEME_CIR_MILSTEIN_TRUNCATED;
    constexpr int S = DEG == 0 ? 1 : (DEG + 2) & ~1;
    constexpr int NB = kLevelBlock;
    extern __shared__ __align__(16) double smd[];
    double *zbuf = smd + v3_table_words(DEG, K1);                         // [kV3Steps][NB]
    uint16_t *list = reinterpret_cast<uint16_t *>(zbuf + kV3Steps * NB);  // tail slots k * NB + t
    __shared__ int tail_cnt[2];
    if constexpr (DEG == 0) {
        for (int i = threadIdx.x; i < K1; i += blockDim.x) smd[i] = __ldg(coeffs + i);
    } else {
        for (int i = threadIdx.x; i < (DEG + 1) * K1; i += blockDim.x) {
            const int d = static_cast<int>(i / K1), j = static_cast<int>(i % K1);
            smd[j * S + d] = __ldg(coeffs + i);
        }
    }
    if (threadIdx.x < 2) tail_cnt[threadIdx.x] = 0;
    const int cap = static_cast<int>(K1 - 1);
    const int t = threadIdx.x, lane = t & 31;
    __shared__ Affine lane_map[NB + 1];  // as k_gaussian_level_v2
    {
        Affine m{1, 0};
        for (int b = 0; b < 8; ++b)
            if ((static_cast<unsigned>(t) >> b) & 1u) m = {A.jump2[b].a * m.a, A.jump2[b].a * m.c + A.jump2[b].c};
        lane_map[t] = m;
        if (t == 0) {
            Affine g{1, 0};
            const uint64_t stride = static_cast<uint64_t>(gridDim.x) * NB;
            for (int b = 0; b < kPathJumpBits; ++b)
                if ((stride >> b) & 1u) g = {A.jump2[b].a * g.a, A.jump2[b].a * g.c + A.jump2[b].c};
            lane_map[NB] = g;
        }
    }
    const int64_t ntiles = (A.path_count + NB - 1) / NB;
    // start state of the CTA's first tile: one thread (of another warp than the
    // stride map's) walks the bits of the path index, the rest read it after the barrier
    __shared__ uint64_t tile_s0;
    if (t == 32) tile_s0 = path_start_state(A, static_cast<uint64_t>(A.path_lo) + static_cast<uint64_t>(blockIdx.x) * NB);
    __syncthreads();
    uint64_t tile_s = tile_s0;
    unsigned blk = 0;  // running block index: selects the tail counter
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t i = tile * NB + t;
        const bool valid = i < A.path_count;
        uint64_t s;
        {
            const Affine my = lane_map[t], nx = lane_map[NB];
            s = my.a * tile_s + my.c;
            tile_s = nx.a * tile_s + nx.c;
        }
        const Affine st = A.step;
        const double x0 = A.x0, dt_f = A.dt_f, dt_c = A.dt_c, sq_f = A.sq_f;
        const double mudt_f = __dmul_rn(A.a, dt_f), mudt_c = __dmul_rn(A.a, dt_c);  // mlmc.py:195
        const double sg = A.b, hs2 = __dmul_rn(__dmul_rn(0.5, A.b), A.b);           // mlmc.py:196-197
        double xf_e = x0, xc_e = x0, xf_a = x0, xc_a = x0;
        auto step = [&](double x, double dw, double dt, double mudt) -> double {
            if constexpr (GBM) {
                double incr = __dadd_rn(mudt, __dmul_rn(sg, dw));
                if (MIL) incr = __dadd_rn(incr, __dmul_rn(hs2, __dsub_rn(__dmul_rn(dw, dw), dt)));
                return __dmul_rn(x, __dadd_rn(1.0, incr));
            } else {
                return cir_step<MIL>(x, dw, dt, A.a, A.b, A.c);
            }
        };
        auto step_e = [&](double x, double dw, double dt, double mudt) -> double {
            if constexpr (GBM && FMA && ARV_GBM_FMA_STEP) {
                double incr = fma(sg, dw, mudt);
                if (MIL) incr = fma(hs2, fma(dw, dw, -dt), incr);
                return fma(x, incr, x);
            } else {
                return step(x, dw, dt, mudt);
            }
        };
        const double sgsq = __dmul_rn(sg, sq_f);  // as k_gaussian_level_v2
        auto step_z = [&](double x, double z, double dt, double mudt) -> double {
            if constexpr (GBM && FMA && ARV_GBM_FMA_STEP && !MIL) return fma(x, fma(sgsq, z, mudt), x);
            else return step_e(x, __dmul_rn(sq_f, z), dt, mudt);
        };
        auto draw = [&]() -> uint32_t {
            const uint32_t w = pcg32_output(s);
            s = st.a * s + st.c;
            return w;
        };
        // phase 1 for N consecutive elements k0 .. k0 + N - 1 (k0 even; N = 4, 2,
        // or 1 for the single last step of an odd fine-step count)
        auto phase1 = [&](auto nconst, int k0, unsigned &pend) {
            constexpr int N = decltype(nconst)::value;
            uint32_t w[N];
            double z[N], a[N];
#pragma unroll
            for (int k = 0; k < N; ++k) w[k] = draw();
            const unsigned pb = g2::central_words<N, FMA>(w, z);
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const double v = g2::reflected(w[k]);
                // a tail element parks +-v: the sign marks the upper tail (v > 0: the sign
                // bit is the complement of w's top bit -- one LOP3 and a predicated second
                // store instead of two 64-bit selects)
                zbuf[(k0 + k) * NB + t] = z[k];
                if ((pb >> k) & 1u)
                    zbuf[(k0 + k) * NB + t] =
                        __hiloint2double(__double2hiint(v) | static_cast<int>(~w[k] & 0x80000000u), __double2loint(v));
                a[k] = g2::table<DEG>(smd, w[k], v, cap, K1);
            }
            pend |= pb << k0;
#pragma unroll
            for (int k = 0; k + 1 < N; k += 2) {  // the approximate side (mlmc.py:216-220)
                xf_a = step(step(xf_a, __dmul_rn(sq_f, a[k]), dt_f, mudt_f), __dmul_rn(sq_f, a[k + 1]), dt_f, mudt_f);
                xc_a = step(xc_a, __dmul_rn(sq_f, __dadd_rn(a[k], a[k + 1])), dt_c, mudt_c);
            }
            if constexpr (N == 1) xf_a = step(xf_a, __dmul_rn(sq_f, a[0]), dt_f, mudt_f);  // mlmc.py:221-226
        };
        for (int64_t k_lo = 0; k_lo < A.n_f; k_lo += kV3Steps) {
            const int L = static_cast<int>(A.n_f - k_lo < kV3Steps ? A.n_f - k_lo : kV3Steps);
            // ---- phase 1
            unsigned pend = 0;
            int k0 = 0;
            for (; k0 + 4 <= L; k0 += 4) phase1(std::integral_constant<int, 4>{}, k0, pend);
            if (k0 + 2 <= L) {
                phase1(std::integral_constant<int, 2>{}, k0, pend);
                k0 += 2;
            }
            if (k0 < L) phase1(std::integral_constant<int, 1>{}, k0, pend);
            {  // append this thread's tail slots to the CTA list
                const int np = __popc(pend);
                int incl = np;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                int base = 0;
                if (lane == 31 && incl) base = atomicAdd(&tail_cnt[blk & 1u], incl);
                base = __shfl_sync(0xffffffffu, base, 31);
                int pos = base + incl - np;
                for (unsigned m = pend; m; m &= m - 1u) {
                    ARV_DCHECK(pos < kV3Steps * NB);
                    list[pos++] = static_cast<uint16_t>((__ffs(m) - 1) * NB + t);
                }
            }
            __syncthreads();
            // ---- phase 2: the CTA serves the whole tail list
            {
                const int nt = tail_cnt[blk & 1u];
                if (t == 0) tail_cnt[(blk + 1u) & 1u] = 0;  // the next block's counter (idle since the last barrier)
                for (int q = t; q < nt; q += NB) {
                    const int slot = list[q];
                    const double pv = zbuf[slot];
                    zbuf[slot] = copysign(g2::tail_abs<FMA, false>(fabs(pv)), pv);  // upper tail positive (exact_dist.py:124-126)
                }
            }
            __syncthreads();
            // ---- phase 3: the exact-side paths, in step order
            int k = 0;
            for (; k + 2 <= L; k += 2) {
                const double z0 = zbuf[k * NB + t], z1 = zbuf[(k + 1) * NB + t];
                xf_e = step_z(step_z(xf_e, z0, dt_f, mudt_f), z1, dt_f, mudt_f);
                xc_e = step_z(xc_e, __dadd_rn(z0, z1), dt_c, mudt_c);
            }
            if (k < L) xf_e = step_z(xf_e, zbuf[k * NB + t], dt_f, mudt_f);
            ++blk;
        }
        double d[ARV_NKIND] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if (valid) {
            const double fe = payoff_fn(xf_e, A.payoff, A.strike);
            const double fa = payoff_fn(xf_a, A.payoff, A.strike);
            const double ce = A.level > 0 ? payoff_fn(xc_e, A.payoff, A.strike) : 0.0;
            const double ca = A.level > 0 ? payoff_fn(xc_a, A.payoff, A.strike) : 0.0;
            d[0] = __dsub_rn(fe, ce);
            d[1] = __dsub_rn(fa, ca);
            d[2] = __dadd_rn(__dsub_rn(__dsub_rn(fe, ce), fa), ca);
            d[3] = fe;
            d[4] = fa;
            if (paths) {
                paths[i] = fe;
                paths[A.path_count + i] = ce;
                paths[2 * A.path_count + i] = fa;
                paths[3 * A.path_count + i] = ca;
            }
        }
        cta_moments<ARV_NKIND>(d, valid, parts + tile * 3 * ARV_NKIND);
    }
}

// Test hook: the level kernels' exact-side normal of each 32-bit word
// (u = (w + 1/2) 2^-32): the FMA central rational, or the tail evaluation
// (neg_log, sqrt_mid, C / D rational) -- the arithmetic k_gaussian_level_v2 /
// _v3 run, element by element.
__global__ void __launch_bounds__(256) k_level_normals(const uint32_t *__restrict__ w, double *__restrict__ out,
                                                       int64_t n) {
    constexpr bool FMA = ARV_GBM_FMA_EXACT != 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t wi[1] = {w[i]};
        double z[1];
        if (g2::central_words<1, FMA>(wi, z)) {
            const double t = g2::tail_abs<FMA, false>(g2::reflected(wi[0]));
            z[0] = wi[0] >> 31 ? t : -t;
        }
        out[i] = z[0];
    }
}

// ----------------------------------------------------------- CIR exact --
// Lambda-sorted transitions.  The exact quantile costs ~3 sweeps whose window
// covers ~16 sqrt(lambda/2) Poisson terms. lambda is proportional to the path
// state, and that state spans an order of magnitude (the CIR law is
// gamma-like). A warp therefore runs as long as its largest-lambda lane: 18-20
// of 32 lanes were active on average. Each step, the CTA first draws the
// uniforms, advances the approximate side and computes the table warm starts
// in path order. It then sorts its 256 exact-side solves by lambda and hands
// them out in sorted order, so each warp solves transitions of similar cost.
// Results return to the owning lane through shared memory. Per-path results
// are unchanged; only the lane that computes them differs. Sorting by the
// predicted sweep length, which also counts the y-dependent part above the
// window, measured 1.7% slower than sorting by lambda. The sort costs 36
// barrier stages per step; config 5 went 68.9 -> 60.6 ms.  Since the
// segmented form below keeps every CTA's lambdas close (grid-wide buckets),
// the per-step sort is only used by the one-kernel form of long levels
// (the SORT instantiation); short levels (<= 8 steps) run faster without it.

// Ascending bitonic sort of (key, slot) over the CTA; perm[t] = slot of rank t.
template <int BS>
__device__ __forceinline__ void cta_sort_perm(double key, double *skey, int *perm) {
    const int t = threadIdx.x;
    skey[t] = key;
    perm[t] = t;
    __syncthreads();
    for (int k = 2; k <= BS; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int o = t ^ j;
            if (o > t) {
                const double a = skey[t], b = skey[o];
                const int ia = perm[t], ib = perm[o];
                const bool gt = a > b || (a == b && ia > ib);
                if (gt == ((t & k) == 0)) {
                    skey[t] = b;
                    skey[o] = a;
                    perm[t] = ib;
                    perm[o] = ia;
                }
            }
            __syncthreads();
        }
    }
}

// Segmented mode (long levels): the level runs as segments of a few steps.
// Between segments the paths are bucketed by lambda over the whole grid
// (counting sort on the float exponent + 3 mantissa bits of lambda, ~9%
// wide buckets), so every CTA holds paths of similar lambda: its warps then
// carry similar sweep lengths and the post-solve barrier stops waiting on
// one heavy warp (28% of warp stall samples in the one-kernel form).  Each
// path's state (both sides, stream position, fail count, path id) travels
// with it in a slot-indexed record; per-path results are unchanged, and the
// statistics are reduced afterwards in path order by the same CTA partition,
// so they are bitwise identical to the one-kernel form.
struct CirSeg {
    int64_t k0, nsteps;
    int first, last;
    const double *xe_in, *xa_in;
    const uint64_t *rs_in;
    const uint32_t *fl_in, *pid_in;
    double *xe_out, *xa_out;
    uint64_t *rs_out;
    uint32_t *fl_out, *pid_out;
    uint32_t *bucket;  // !last: lambda bucket of each slot's next step
    uint32_t *hist;    // !last: global bucket counts (zeroed by the caller)
    double *pay;       // last (segmented): pay[pid] = p_exact, pay[n + pid] = p_approx
};
constexpr int kCirBuckets = 256;

__device__ __forceinline__ uint32_t cir_bucket(double lam) {
    // lambda in [2^-8, 2^24) -> 8 buckets per octave; clamped outside
    const int b = static_cast<int>(__float_as_uint(static_cast<float>(lam)) >> 20) - ((127 - 8) << 3);
    return static_cast<uint32_t>(b < 0 ? 0 : (b >= kCirBuckets ? kCirBuckets - 1 : b));
}

template <int DEG, bool SORT>
__global__ void __launch_bounds__(kCirBlock, ARV_CIR_MINB) k_cir_exact_level(LevelArgs A, const double *__restrict__ stacks,
                                                                 int64_t n_knots, int64_t K1, int use_smem,
                                                                 double *__restrict__ parts,
                                                                 double *__restrict__ paths,
                                                                 unsigned long long *__restrict__ n_fail, CirSeg G) {
    extern __shared__ double smd[];
    const double *tab = stacks;
    if (use_smem) {
        double *st = smd;
        const int64_t total = 2 * n_knots * (DEG + 1) * K1;
        for (int64_t k = threadIdx.x; k < total; k += blockDim.x) st[k] = __ldg(stacks + k);
        __syncthreads();
        tab = st;
    }
    // The path this thread owns (slot i): its stream, both states and fail
    // count.  The exact solve of a step may run on another lane of the CTA
    // (the SORT instantiation).
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = i < A.path_count;
    uint32_t pid = static_cast<uint32_t>(valid ? i : 0);
    double x_e = A.x0, x_a = A.x0;
    unsigned fails = 0;
    if (!G.first && valid) {
        pid = G.pid_in[i];
        x_e = G.xe_in[i];
        x_a = G.xa_in[i];
        fails = G.fl_in[i];
    }
    PathRng rng(A, static_cast<uint64_t>(A.path_lo + pid), G.first || !valid ? nullptr : G.rs_in + i);
    __shared__ double sh_key[SORT ? kCirBlock : 1], sh_u[SORT ? kCirBlock : 1], sh_lam[SORT ? kCirBlock : 1],
        sh_warm[SORT ? kCirBlock : 1], sh_x[SORT ? kCirBlock : 1], sh_r[SORT ? kCirBlock : 1];
    __shared__ int sh_perm[SORT ? kCirBlock : 1];
    for (int64_t k = 0; k < G.nsteps; ++k) {
        double u = 0.5, lam_e = 0.0, warm = 0.0;
        if (valid) {
            u = rng.next();
            // mlmc.py:264-268 approximate side (state clamped before lambda)
            const double lam_a = __dmul_rn(fmax(x_a, 0.0), A.decay_over_scale);
            x_a = __dmul_rn(A.scale, ncchi2_eval1<DEG>(tab, n_knots, K1, A.nu_table, u, lam_a));
            // mlmc.py:269-278 exact side, warm-started from the table
            lam_e = __dmul_rn(x_e, A.decay_over_scale);
            if (A.want_exact) warm = ncchi2_warm1<DEG>(tab, n_knots, K1, A.nu_table, u, lam_e);
        }
        if constexpr (SORT) {
            const int t = threadIdx.x;
            cta_sort_perm<kCirBlock>(valid && A.want_exact ? lam_e : -1.0, sh_key, sh_perm);
            sh_u[t] = u;
            sh_lam[t] = lam_e;
            sh_warm[t] = warm;
            __syncthreads();
            const int src = sh_perm[t];  // solve the transition of rank t
            const bool solve = sh_key[t] >= 0.0;
            double xq = 0.0, rq = 0.0;
            if (solve) {
                const NcQuantile q = ncchi2_quantile(sh_u[src], A.nu_exact, sh_lam[src], sh_warm[src]);
                xq = q.x;
                rq = q.resid;
            }
            sh_x[src] = xq;  // back to the owner's slot
            sh_r[src] = rq;
            __syncthreads();
            if (valid && A.want_exact) {
                fails += sh_r[t] > 1e-8;
                x_e = __dmul_rn(A.scale, sh_x[t]);
            }
            __syncthreads();
        } else if (valid && A.want_exact) {
            const NcQuantile q = ncchi2_quantile(u, A.nu_exact, lam_e, warm);
            fails += q.resid > 1e-8;
            x_e = __dmul_rn(A.scale, q.x);
        }
    }
    if (!G.last) {  // hand the record on and count its next-step lambda bucket
        __shared__ uint32_t hist[kCirBuckets];
        for (int b = threadIdx.x; b < kCirBuckets; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        if (valid) {
            G.xe_out[i] = x_e;
            G.xa_out[i] = x_a;
            G.rs_out[i] = rng.s;
            G.fl_out[i] = fails;
            G.pid_out[i] = pid;
            const uint32_t b = cir_bucket(__dmul_rn(x_e, A.decay_over_scale));
            G.bucket[i] = b;
            ARV_DCHECK(b < kCirBuckets);
            atomicAdd(&hist[b], 1u);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < kCirBuckets; b += blockDim.x)
            if (hist[b]) atomicAdd(&G.hist[b], hist[b]);
        return;
    }
    const double fe = payoff_fn(x_e, A.payoff, A.strike);
    const double fa = payoff_fn(x_a, A.payoff, A.strike);
    if (valid && fails && n_fail) atomicAdd(n_fail, static_cast<unsigned long long>(fails));
    if (!G.first) {  // segmented: payoffs by path id, reduced in path order afterwards
        if (valid) {
            G.pay[pid] = fe;
            G.pay[A.path_count + pid] = fa;
        }
        return;
    }
    double d[ARV_NKIND] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (valid) {
        // coarse slots repeat the fine payoffs (mlmc.py:281-286), so both
        // two-way differences vanish; slot 2 carries the exact - approx
        // correction of reproduce.py:299-301, slots 3/4 the process values.
        d[2] = __dsub_rn(fe, fa);
        d[3] = fe;
        d[4] = fa;
        if (paths) {
            paths[i] = fe;
            paths[A.path_count + i] = fe;  // coarse slots repeat fine (mlmc.py:281-286)
            paths[2 * A.path_count + i] = fa;
            paths[3 * A.path_count + i] = fa;
        }
    }
    cta_moments<ARV_NKIND, kCirBlock>(d, valid, parts + static_cast<int64_t>(blockIdx.x) * 3 * ARV_NKIND);
}

// Exclusive scan of the bucket counts into per-bucket cursors; clears the
// counts for the next segment.  One CTA of kCirBuckets threads.
__global__ void __launch_bounds__(kCirBuckets) k_cir_bucket_scan(uint32_t *hist, uint32_t *cursor) {
    __shared__ uint32_t sh[kCirBuckets];
    const int t = threadIdx.x;
    const uint32_t v = hist[t];
    sh[t] = v;
    __syncthreads();
    for (int o = 1; o < kCirBuckets; o <<= 1) {  // Hillis-Steele inclusive scan
        const uint32_t add = t >= o ? sh[t - o] : 0u;
        __syncthreads();
        sh[t] += add;
        __syncthreads();
    }
    cursor[t] = sh[t] - v;
    hist[t] = 0;
}

// Move each record to its bucket's range (a CTA reserves one contiguous run
// per bucket it holds; order inside a bucket is immaterial to the results).
__global__ void __launch_bounds__(kCirBlock) k_cir_scatter(int64_t n, const uint32_t *__restrict__ bucket,
                                                           uint32_t *cursor, const double *__restrict__ xe,
                                                           const double *__restrict__ xa,
                                                           const uint64_t *__restrict__ rs,
                                                           const uint32_t *__restrict__ fl,
                                                           const uint32_t *__restrict__ pid, double *xe_o,
                                                           double *xa_o, uint64_t *rs_o, uint32_t *fl_o,
                                                           uint32_t *pid_o) {
    __shared__ uint32_t cnt[kCirBuckets], base[kCirBuckets];
    for (int b = threadIdx.x; b < kCirBuckets; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t b = 0, local = 0;
    if (i < n) {
        b = bucket[i];
        local = atomicAdd(&cnt[b], 1u);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kCirBuckets; c += blockDim.x)
        if (cnt[c]) base[c] = atomicAdd(&cursor[c], cnt[c]);
    __syncthreads();
    if (i < n) {
        const uint32_t dst = base[b] + local;
        ARV_DCHECK(b < kCirBuckets && dst < static_cast<uint64_t>(n));
        xe_o[dst] = xe[i];
        xa_o[dst] = xa[i];
        rs_o[dst] = rs[i];
        fl_o[dst] = fl[i];
        pid_o[dst] = pid[i];
    }
}

// Statistics of a segmented level, in path order with the one-kernel CTA
// partition (bitwise identical to it).
__global__ void __launch_bounds__(kCirBlock) k_cir_payoff_moments(LevelArgs A, const double *__restrict__ pay,
                                                                  double *__restrict__ parts,
                                                                  double *__restrict__ paths) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = i < A.path_count;
    double d[ARV_NKIND] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (valid) {
        const double fe = pay[i], fa = pay[A.path_count + i];
        d[2] = __dsub_rn(fe, fa);
        d[3] = fe;
        d[4] = fa;
        if (paths) {
            paths[i] = fe;
            paths[A.path_count + i] = fe;
            paths[2 * A.path_count + i] = fa;
            paths[3 * A.path_count + i] = fa;
        }
    }
    cta_moments<ARV_NKIND, kCirBlock>(d, valid, parts + static_cast<int64_t>(blockIdx.x) * 3 * ARV_NKIND);
}

// -------------------------------------------------- standalone ncchi2 --
// Per-element lambda: tiles of 256 elements are solved in lambda order (the
// sort of the CIR level kernel) so that a warp's lanes have similar window
// lengths; a shared lambda needs no sort.
__global__ void __launch_bounds__(kLevelBlock) k_ncchi2_inv(const double *__restrict__ u, const double *__restrict__ lam,
                                                            int64_t nlam, double nu, const double *__restrict__ x0,
                                                            double tol, double *__restrict__ out,
                                                            double *__restrict__ resid, int64_t n) {
    if (nlam == 1) {
        const double l0 = lam[0];
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const NcQuantile q = ncchi2_quantile(u[i], nu, l0, x0 ? x0[i] : -1.0, tol);
            out[i] = q.x;
            if (resid) resid[i] = q.resid;
        }
        return;
    }
    __shared__ double sh_key[kLevelBlock];
    __shared__ int sh_perm[kLevelBlock];
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * kLevelBlock; base < n;
         base += static_cast<int64_t>(gridDim.x) * kLevelBlock) {  // CTA-uniform tile loop
        const int64_t mine = base + threadIdx.x;
        cta_sort_perm<kLevelBlock>(mine < n ? lam[mine] : -1.0, sh_key, sh_perm);
        const int64_t i = base + sh_perm[threadIdx.x];  // element of rank t (tail slots sort first)
        if (i < n) {
            const NcQuantile q = ncchi2_quantile(u[i], nu, lam[i], x0 ? x0[i] : -1.0, tol);
            out[i] = q.x;
            if (resid) resid[i] = q.resid;
        }
        __syncthreads();  // sh_key / sh_perm reused by the next tile
    }
}
__global__ void __launch_bounds__(256) k_ncchi2_cdf(const double *__restrict__ x, const double *__restrict__ lam,
                                                    int64_t nlam, double nu, double *__restrict__ out, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double li = nlam == 1 ? lam[0] : lam[i];
        const double xi = x[i];
        out[i] = xi <= 0.0 ? 0.0 : ncchi2_cdf_minus(0.5 * nu, xi, nc_lam(li), 0.0).resid;
    }
}

// ---------------------------------------------------------------- host --
static int fill_common(const arv_level_spec *sp, LevelArgs &A) {
    if (!sp) return set_error(ARV_ERR_CONFIG, "null level spec");
    if (sp->level < 0) return set_error(ARV_ERR_CONFIG, "level must be >= 0");
    if (sp->n0 < 1) return set_error(ARV_ERR_CONFIG, "n0 must be >= 1");
    if (sp->payoff != ARV_PAYOFF_IDENTITY && sp->payoff != ARV_PAYOFF_CALL)
        return set_error(ARV_ERR_CONFIG, "unknown payoff %d", sp->payoff);
    if (sp->path_count < 0 || sp->path_lo < 0 || sp->path_lo + sp->path_count > sp->n_paths_total)
        return set_error(ARV_ERR_CONFIG, "path range [%lld, +%lld) outside n_paths_total=%lld", (long long)sp->path_lo,
                         (long long)sp->path_count, (long long)sp->n_paths_total);
    if (sp->level > 40) return set_error(ARV_ERR_CONFIG, "level too large");
    A.a = sp->a;
    A.b = sp->b;
    A.c = sp->c;
    A.x0 = sp->x0;
    A.strike = sp->strike;
    A.level = sp->level;
    A.payoff = sp->payoff;
    A.n_f = static_cast<int64_t>(sp->n0) << sp->level;
    A.dt_f = sp->t_end / static_cast<double>(A.n_f);  // mlmc.py:119-120
    A.dt_c = 2.0 * A.dt_f;
    A.sq_f = std::sqrt(A.dt_f);
    const StreamStart st = pcg32_start(sp->seed, sp->stream_id, 0);
    A.s0 = st.state;
    A.inc = st.inc;
    A.step = lcg_jump(static_cast<uint64_t>(sp->n_paths_total), st.inc);
    Affine j2 = lcg_jump(1, st.inc);
    for (int b = 0; b < kPathJumpBits; ++b) {
        A.jump2[b] = j2;
        j2 = {j2.a * j2.a, j2.a * j2.c + j2.c};  // compose the map with itself
    }
    if (static_cast<uint64_t>(sp->n_paths_total) >> kPathJumpBits)
        return set_error(ARV_ERR_CONFIG, "n_paths_total must be < 2^40");
    if (sp->rng != ARV_RNG_PCG32 && sp->rng != ARV_RNG_PHILOX) return set_error(ARV_ERR_CONFIG, "unknown rng %d", sp->rng);
    A.rng = sp->rng;
    if (sp->sides < ARV_SIDES_BOTH || sp->sides > ARV_SIDES_APPROX)
        return set_error(ARV_ERR_CONFIG, "unknown sides %d", sp->sides);
    A.want_exact = sp->sides != ARV_SIDES_APPROX;
    A.want_approx = sp->sides != ARV_SIDES_EXACT;
    A.seed = sp->seed;
    A.sid = sp->stream_id;
    A.n_paths_total = static_cast<uint64_t>(sp->n_paths_total);
    A.path_lo = sp->path_lo;
    A.path_count = sp->path_count;
    A.nu_exact = A.nu_table = A.scale = A.decay_over_scale = 0.0;
    return ARV_OK;
}

static int64_t n_blocks_for(int64_t count, int bs = kLevelBlock) { return (count + bs - 1) / bs; }

static int run_finalize(double *parts, int64_t nb, double *stats, cudaStream_t s, const char *what,
                        FinScratch *fs = nullptr) {
    if (!fs || nb <= kFinSingleMax) {
        k_finalize<ARV_NKIND><<<1, kFinalBlock, 0, s>>>(parts, nb, stats);
        note_launch();
        return check_launch(what);
    }
    cudaMemsetAsync(&fs->ticket, 0, sizeof(unsigned), s);
    k_finalize_chunks<ARV_NKIND><<<kFinChunks, kFinStageBlock, 0, s>>>(parts, nb, fs, stats);
    note_launch();
    return check_launch(what);
}

// Steps per segment of a segmented CIR exact level (0: always one kernel);
// arv_set_tuning(ARV_TUNE_CIR_SEGMENT).
int g_cir_segment = 4;
// Gaussian level kernel for both-sides PCG32 levels: 0 = default, 2 or 3;
// arv_set_tuning(ARV_TUNE_GBM_KERNEL) (tests compare the two bit for bit).
int g_gbm_kernel = 0;

static int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

// Chunked-finalize scratch after nb CTA partials in a caller workspace, or
// nullptr when the workspace holds only the partials (older callers).
static FinScratch *fin_scratch(void *ws, int64_t ws_bytes, int64_t nb) {
    const int64_t off = align256(nb * 3 * ARV_NKIND * int64_t(sizeof(double)));
    return ws_bytes >= off + int64_t(sizeof(FinScratch)) ? reinterpret_cast<FinScratch *>(static_cast<char *>(ws) + off)
                                                          : nullptr;
}

// Workspace of a segmented CIR exact level: CTA partials, two record
// buffers (slot-indexed SoA), buckets, bucket counts / cursors, payoffs.
struct CirWs {
    int64_t total = 0;
    double *parts = nullptr, *xe[2] = {}, *xa[2] = {}, *pay = nullptr;
    uint64_t *rs[2] = {};
    uint32_t *fl[2] = {}, *pid[2] = {}, *bucket = nullptr, *hist = nullptr, *cursor = nullptr;
    FinScratch *fin = nullptr;
    CirWs(int64_t n, void *base) {
        char *p = static_cast<char *>(base);
        auto take = [&](int64_t bytes) -> void * {
            void *r = p ? p + total : nullptr;
            total += align256(bytes);
            return r;
        };
        parts = static_cast<double *>(take(n_blocks_for(n, kCirBlock) * 3 * ARV_NKIND * int64_t(sizeof(double))));
        for (int b = 0; b < 2; ++b) {
            xe[b] = static_cast<double *>(take(8 * n));
            xa[b] = static_cast<double *>(take(8 * n));
            rs[b] = static_cast<uint64_t *>(take(8 * n));
            fl[b] = static_cast<uint32_t *>(take(4 * n));
            pid[b] = static_cast<uint32_t *>(take(4 * n));
        }
        bucket = static_cast<uint32_t *>(take(4 * n));
        hist = static_cast<uint32_t *>(take(4 * kCirBuckets));
        cursor = static_cast<uint32_t *>(take(4 * kCirBuckets));
        pay = static_cast<double *>(take(16 * n));
        fin = static_cast<FinScratch *>(take(sizeof(FinScratch)));
    }
};

}  // namespace arv

namespace arv {
int set_nc_certify(int on) {
    const int v = on ? 1 : 0;
    cudaMemcpyToSymbol(g_nc_certify_on, &v, sizeof v);
    return check_launch("arv_set_tuning(ARV_TUNE_NC_CERTIFY)");
}
}  // namespace arv

using namespace arv;

extern "C" {

int64_t arv_mlmc_workspace_bytes(int64_t path_count) {
    const int64_t nb = n_blocks_for(path_count < 1 ? 1 : path_count, kMinLevelBlock);
    return align256(nb * 3 * ARV_NKIND * static_cast<int64_t>(sizeof(double))) + int64_t(sizeof(FinScratch));
}

int64_t arv_mlmc_cir_workspace_bytes(int64_t path_count) {
    return CirWs(path_count < 1 ? 1 : path_count, nullptr).total;
}

// Raise a kernel's dynamic shared-memory limit (static + dynamic may pass
// the 48 KB default) once per kernel and size.
static void allow_dyn_smem(const void *fn, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void *, size_t>> done;
    std::lock_guard<std::mutex> lock(mu);
    for (auto &e : done)
        if (e.first == fn && e.second >= bytes) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    done.emplace_back(fn, bytes);
}

// one wave of resident CTAs (at most one per tile)
#ifndef ARV_GBM_V2_WAVES
#define ARV_GBM_V2_WAVES 8  // waves of the grid: 1 -> 5.97 ms at level 8, 2 -> 5.69, 8 -> 5.55 (dynamic CTA scheduling still pays)
#endif
static unsigned grid_v2(const void *fn, int64_t tiles, size_t smem) {
    const int64_t wave = static_cast<int64_t>(resident_ctas(fn, kLevelBlock, smem)) * device_sm_count() * ARV_GBM_V2_WAVES;
    return static_cast<unsigned>(tiles < wave ? tiles : wave);
}

int arv_mlmc_gaussian_level(const arv_level_spec *spec, const double *coeffs, int degree, int64_t K1, double *stats,
                            double *paths, void *workspace, int64_t workspace_bytes, void *stream) {
    LevelArgs A;
    if (int rc = fill_common(spec, A)) return rc;
    const int scheme = spec->scheme;
    if (scheme == ARV_SCHEME_EM || scheme == ARV_SCHEME_MILSTEIN) {
        if (!(spec->b > 0 && spec->x0 > 0 && spec->t_end > 0))
            return set_error(ARV_ERR_CONFIG, "GBM requires sigma > 0, x0 > 0, t_end > 0");
    } else if (scheme == ARV_SCHEME_CIR_EULER_TRUNCATED || scheme == ARV_SCHEME_CIR_MILSTEIN_TRUNCATED) {
        if (!(spec->a > 0 && spec->b > 0 && spec->c > 0 && spec->x0 > 0 && spec->t_end > 0))
            return set_error(ARV_ERR_CONFIG, "CIR requires kappa, theta, sigma, x0, t_end > 0");
    } else {
        return set_error(ARV_ERR_CONFIG, "arv_mlmc_gaussian_level cannot run scheme %d", scheme);
    }
    // degree 0: piecewise-constant table values[K1]; >= 1: dyadic (degree+1, K1)
    if (K1 < 2 || sizeof(double) * (degree + 1) * K1 > 48 * 1024)
        return set_error(ARV_ERR_CONFIG, "table size out of range (degree %d, %lld columns)", degree, (long long)K1);
    if (spec->path_count < 1) return set_error(ARV_ERR_CONFIG, "need at least one path");
    const int64_t nb = n_blocks_for(spec->path_count);
    if (workspace_bytes < nb * 3 * ARV_NKIND * static_cast<int64_t>(sizeof(double)))
        return set_error(ARV_ERR_CONFIG, "workspace too small");
    double *parts = static_cast<double *>(workspace);
    const size_t smem = sizeof(double) * (degree + 1) * K1;
    // v2 table layout: interleaved [K1][S], S = degree + 1 rounded up to even
    const size_t smem2 = sizeof(double) * (degree == 0 ? 1 : ((degree + 2) & ~1)) * K1;
    // v3 (phased exact side): both sides wanted, PCG32; the table + the block buffers
    const size_t smem3 = v3_smem_bytes(degree, K1);
    // auto: the phased kernel from 8 fine steps per path on; below that its per-block machinery (two
    // barriers, the CTA-wide tail list) costs more than it saves (levels 0 / 1 / 2 of config 4: 0.101 /
    // 0.116 / 0.142 ms with v2 against 0.121 / 0.129 / 0.152 ms; level 3 ties).  Same results bit for bit.
    const int kern = g_gbm_kernel ? g_gbm_kernel : (ARV_GBM_V3 && A.n_f >= 8 ? 3 : 2);
    const bool use_v3 = kern == 3 && A.rng == ARV_RNG_PCG32 && A.want_exact && A.want_approx &&
                        smem3 <= 96 * 1024;
    cudaStream_t s = as_stream(stream);
#define ARV_LAUNCH(D, S)                                                                              \
    (A.rng == ARV_RNG_PHILOX                                                                          \
         ? k_gaussian_level<D, S, true><<<(unsigned)nb, kLevelBlock, smem, s>>>(A, coeffs, K1, parts, paths) \
         : (use_v3 ? k_gaussian_level_v3<D, S><<<grid_v2((const void *)k_gaussian_level_v3<D, S>, nb, smem3), \
                                                 kLevelBlock, smem3, s>>>(A, coeffs, K1, parts, paths)                     \
         : (ARV_GBM_V2 ? ((A.want_exact && A.want_approx && ARV_GBM_SIDES_SPLIT)                         \
                              ? k_gaussian_level_v2<D, S, true><<<grid_v2((const void *)k_gaussian_level_v2<D, S, true>, nb, smem2), \
                                                                  kLevelBlock, smem2, s>>>(A, coeffs, K1, parts, paths) \
                              : k_gaussian_level_v2<D, S, false><<<grid_v2((const void *)k_gaussian_level_v2<D, S, false>, nb, smem2), \
                                                                   kLevelBlock, smem2, s>>>(A, coeffs, K1, parts, paths)) \
                       : k_gaussian_level<D, S, false><<<(unsigned)nb, kLevelBlock, smem, s>>>(A, coeffs, K1, parts, paths))))
#define ARV_V3_ATTR(D, S) \
    if (use_v3) allow_dyn_smem((const void *)k_gaussian_level_v3<D, S>, smem3);
#define ARV_SCHEMES(D)                                                                      \
    case D:                                                                                 \
        switch (scheme) {                                                                   \
            case ARV_SCHEME_EM: ARV_V3_ATTR(D, ARV_SCHEME_EM) ARV_LAUNCH(D, ARV_SCHEME_EM); break; \
            case ARV_SCHEME_MILSTEIN: ARV_V3_ATTR(D, ARV_SCHEME_MILSTEIN) ARV_LAUNCH(D, ARV_SCHEME_MILSTEIN); break; \
            case ARV_SCHEME_CIR_EULER_TRUNCATED: ARV_V3_ATTR(D, ARV_SCHEME_CIR_EULER_TRUNCATED)             \
                ARV_LAUNCH(D, ARV_SCHEME_CIR_EULER_TRUNCATED); break;                       \
            default: ARV_V3_ATTR(D, ARV_SCHEME_CIR_MILSTEIN_TRUNCATED)                      \
                ARV_LAUNCH(D, ARV_SCHEME_CIR_MILSTEIN_TRUNCATED); break;                    \
        }                                                                                   \
        break;
    switch (degree) {
        ARV_SCHEMES(0)
        ARV_SCHEMES(1)
        ARV_SCHEMES(2)
        ARV_SCHEMES(3)
        ARV_SCHEMES(4)
        ARV_SCHEMES(5)
        default: return set_error(ARV_ERR_CONFIG, "table degree must be in [0, 5], got %d", degree);
    }
#undef ARV_SCHEMES
#undef ARV_LAUNCH
#undef ARV_V3_ATTR
    note_launch();
    if (int rc = check_launch("arv_mlmc_gaussian_level")) return rc;
    return run_finalize(parts, nb, stats, s, "arv_mlmc_gaussian_level(finalize)",
                        fin_scratch(workspace, workspace_bytes, nb));
}

int arv_mlmc_cir_exact_level(const arv_level_spec *spec, const double *stacks, int64_t n_knots, int degree, int64_t K1,
                             double nu, double *stats, double *paths, int64_t *n_fail, void *workspace,
                             int64_t workspace_bytes, void *stream) {
    LevelArgs A;
    if (int rc = fill_common(spec, A)) return rc;
    if (spec->scheme != ARV_SCHEME_CIR_EXACT) return set_error(ARV_ERR_CONFIG, "cir_exact level needs scheme CIR_EXACT");
    const double kappa = spec->a, theta = spec->b, sigma = spec->c;
    if (!(kappa > 0 && theta > 0 && sigma > 0 && spec->x0 > 0 && spec->t_end > 0))
        return set_error(ARV_ERR_CONFIG, "CIR requires kappa, theta, sigma, x0, t_end > 0");
    if (!(nu > 0)) return set_error(ARV_ERR_CONFIG, "nu must be > 0");
    if (n_knots < 2 || K1 < 2) return set_error(ARV_ERR_CONFIG, "bad ncchi2 table shape");
    if (spec->path_count < 1) return set_error(ARV_ERR_CONFIG, "need at least one path");
    // exact_dist.py:561-564 (cir_transition_params) and mlmc.py:254-257
    const double dt = A.dt_f;
    const double decay = std::exp(-kappa * dt);
    A.scale = sigma * sigma * (1.0 - decay) / (4.0 * kappa);
    A.nu_exact = 4.0 * kappa * theta / (sigma * sigma);
    A.decay_over_scale = std::exp(-kappa * dt) / A.scale;
    A.nu_table = nu;
    const int64_t n = spec->path_count;
    const int64_t nb = n_blocks_for(n, kCirBlock);
    if (workspace_bytes < nb * 3 * ARV_NKIND * static_cast<int64_t>(sizeof(double)))
        return set_error(ARV_ERR_CONFIG, "workspace too small");
    const size_t bytes = sizeof(double) * 2 * n_knots * (degree + 1) * K1;
    const int use_smem = bytes <= 128 * 1024;
    const size_t smem = use_smem ? bytes : 0;
    cudaStream_t s = as_stream(stream);
    unsigned long long *nf = reinterpret_cast<unsigned long long *>(n_fail);
    // Segmented when the level is longer than one segment, the path ids fit
    // 32 bits and the caller's workspace holds the records.
    const int64_t seg = g_cir_segment;
    const bool segmented = seg > 0 && A.want_exact && A.n_f > seg && n < (int64_t(1) << 32) &&
                           workspace_bytes >= CirWs(n, nullptr).total;
    const CirWs W(n, workspace);
    double *parts = segmented ? W.parts : static_cast<double *>(workspace);
    // CTA lambda sort per step: only for the one-kernel form of long levels
    const bool sort = !segmented && A.n_f > 8;
    const void *fn = nullptr;
#define ARV_PICK(D) fn = sort ? (const void *)k_cir_exact_level<D, true> : (const void *)k_cir_exact_level<D, false>
    switch (degree) {
        case 1: ARV_PICK(1); break;
        case 2: ARV_PICK(2); break;
        case 3: ARV_PICK(3); break;
        case 4: ARV_PICK(4); break;
        case 5: ARV_PICK(5); break;
        default: return set_error(ARV_ERR_CONFIG, "polynomial degree must be in [1, 5], got %d", degree);
    }
#undef ARV_PICK
    if (smem > 40 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    auto launch = [&](const CirSeg &G) {
        void *args[] = {(void *)&A, (void *)&stacks, (void *)&n_knots, (void *)&K1, (void *)&use_smem,
                        (void *)&parts, (void *)&paths, (void *)&nf, (void *)&G};
        cudaLaunchKernel(fn, dim3((unsigned)nb), dim3(kCirBlock), args, smem, s);
        note_launch();
    };
    if (!segmented) {
        CirSeg G{};
        G.k0 = 0;
        G.nsteps = A.n_f;
        G.first = G.last = 1;
        launch(G);
        if (int rc = check_launch("arv_mlmc_cir_exact_level")) return rc;
        return run_finalize(parts, nb, stats, s, "arv_mlmc_cir_exact_level(finalize)",
                            fin_scratch(workspace, workspace_bytes, nb));
    }
    cudaMemsetAsync(W.hist, 0, 4 * kCirBuckets, s);
    for (int64_t k0 = 0; k0 < A.n_f; k0 += seg) {
        CirSeg G{};
        G.k0 = k0;
        G.nsteps = A.n_f - k0 < seg ? A.n_f - k0 : seg;
        G.first = k0 == 0;
        G.last = k0 + G.nsteps >= A.n_f;
        G.xe_in = W.xe[0];
        G.xa_in = W.xa[0];
        G.rs_in = W.rs[0];
        G.fl_in = W.fl[0];
        G.pid_in = W.pid[0];
        G.xe_out = W.xe[1];
        G.xa_out = W.xa[1];
        G.rs_out = W.rs[1];
        G.fl_out = W.fl[1];
        G.pid_out = W.pid[1];
        G.bucket = W.bucket;
        G.hist = W.hist;
        G.pay = W.pay;
        launch(G);
        if (int rc = check_launch("arv_mlmc_cir_exact_level(segment)")) return rc;
        if (G.last) break;
        k_cir_bucket_scan<<<1, kCirBuckets, 0, s>>>(W.hist, W.cursor);
        note_launch();
        k_cir_scatter<<<(unsigned)nb, kCirBlock, 0, s>>>(n, W.bucket, W.cursor, W.xe[1], W.xa[1], W.rs[1], W.fl[1],
                                                          W.pid[1], W.xe[0], W.xa[0], W.rs[0], W.fl[0], W.pid[0]);
        note_launch();
        if (int rc = check_launch("arv_mlmc_cir_exact_level(rebucket)")) return rc;
    }
    k_cir_payoff_moments<<<(unsigned)nb, kCirBlock, 0, s>>>(A, W.pay, parts, paths);
    note_launch();
    if (int rc = check_launch("arv_mlmc_cir_exact_level(moments)")) return rc;
    return run_finalize(parts, nb, stats, s, "arv_mlmc_cir_exact_level(finalize)", W.fin);
}

int arv_ncchi2_inv_cdf_tol(const double *u, const double *lam, int64_t nlam, double nu, const double *x0, double tol,
                           double *out, double *resid, int64_t n, void *stream) {
    if (!(nu > 0)) return set_error(ARV_ERR_DOMAIN, "degrees of freedom must be > 0");
    if (!(tol > 0)) return set_error(ARV_ERR_CONFIG, "tolerance must be > 0");
    if (nlam != 1 && nlam != n) return set_error(ARV_ERR_CONFIG, "per-element lambda must match the shape of u");
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_ncchi2_inv<<<stream_grid(n, kLevelBlock, 8), kLevelBlock, 0, as_stream(stream)>>>(u, lam, nlam, nu, x0, tol, out,
                                                                                       resid, n);
    note_launch();
    return check_launch("arv_ncchi2_inv_cdf");
}

int arv_ncchi2_inv_cdf(const double *u, const double *lam, int64_t nlam, double nu, const double *x0, double *out,
                       double *resid, int64_t n, void *stream) {
    return arv_ncchi2_inv_cdf_tol(u, lam, nlam, nu, x0, 1e-9, out, resid, n, stream);
}

int arv_ncchi2_cdf(const double *x, const double *lam, int64_t nlam, double nu, double *out, int64_t n, void *stream) {
    if (!(nu > 0)) return set_error(ARV_ERR_DOMAIN, "degrees of freedom must be > 0");
    if (nlam != 1 && nlam != n) return set_error(ARV_ERR_CONFIG, "per-element lambda must match the shape of x");
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_ncchi2_cdf<<<stream_grid(n, 256, 8), 256, 0, as_stream(stream)>>>(x, lam, nlam, nu, out, n);
    note_launch();
    return check_launch("arv_ncchi2_cdf");
}

int arv_test_level_normals(const uint32_t *words, double *out, int64_t n, void *stream) {
    if (n <= 0) return n < 0 ? set_error(ARV_ERR_CONFIG, "negative n") : ARV_OK;
    k_level_normals<<<stream_grid(n, 256, 8), 256, 0, as_stream(stream)>>>(words, out, n);
    note_launch();
    return check_launch("arv_test_level_normals");
}

// Quantile solves that took the certified single-sweep shortcut since the last call (and reset).
ARV_API int arv_nc_certified_count(unsigned long long *out) {
    if (!out) return set_error(ARV_ERR_CONFIG, "arv_nc_certified_count: null output");
    cudaMemcpyFromSymbol(out, g_nc_certified, sizeof(unsigned long long));
    const unsigned long long zero = 0;
    cudaMemcpyToSymbol(g_nc_certified, &zero, sizeof zero);
    return check_launch("arv_nc_certified_count");
}

#if ARV_NC_COUNT
// diagnostic build only: {CDF evaluations, quantile solves} since the last call
// out[0..1] = evaluations, solves; out[2..9] per-solve histogram; out[10..17] per-warp-max histogram
ARV_API int arv_nc_counters(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_nc_evals, sizeof(unsigned long long));
    cudaMemcpyFromSymbol(out + 1, g_nc_solves, sizeof(unsigned long long));
    cudaMemcpyFromSymbol(out + 2, g_nc_hist, 8 * sizeof(unsigned long long));
    cudaMemcpyFromSymbol(out + 10, g_nc_warp_hist, 8 * sizeof(unsigned long long));
    const unsigned long long zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_nc_evals, zero, sizeof(unsigned long long));
    cudaMemcpyToSymbol(g_nc_solves, zero, sizeof(unsigned long long));
    cudaMemcpyToSymbol(g_nc_hist, zero, sizeof zero);
    cudaMemcpyToSymbol(g_nc_warp_hist, zero, sizeof zero);
    return check_launch("arv_nc_counters");
}
#endif

}  // extern "C"

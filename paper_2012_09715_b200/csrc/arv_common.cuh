// Shared device helpers: PCG32 (state in registers, affine jump-ahead),
// the integer-domain uniform mapping, the AS241 rational, launch helpers and
// the per-thread error slot behind arv_last_error().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cassert>
#include <cstdio>
#include <string>

#include "approxrv_b200.h"

// Device-side bounds / invariant checks for the checked build
// (-DARV_CHECKS=1, tools/build_checked.py): compute-sanitizer is closed on the
// GPU pool, so the risky indices (warp tail lists, CIR bucket scatter, table
// indices, finalize tickets) assert their ranges instead and the GPU test
// suite runs against that library.  Compiled out otherwise.
#ifndef ARV_CHECKS
#define ARV_CHECKS 0
#endif
#if ARV_CHECKS
#define ARV_DCHECK(c) assert(c)
#else
#define ARV_DCHECK(c) ((void)0)
#endif

namespace arv {

constexpr uint64_t kPcgMult = 6364136223846793005ULL;
constexpr int kNumSMs = 148;  // B200; the launcher queries the device anyway

// ---------------------------------------------------------------- errors --
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);
void note_launch(int n = 1);
int device_sm_count();
// Resident CTAs per SM of `fn` at this block size and dynamic smem (occupancy
// calculator, cached per kernel / shape / device).
int resident_ctas(const void *fn, int block, size_t smem);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ----------------------------------------------------------------- PCG32 --
struct Affine {
    uint64_t a, c;  // s -> a*s + c (mod 2^64)
};

// Jump-ahead of the LCG s' = M s + inc by `delta` steps (square-and-multiply
// on the affine map; O(log delta)).
__host__ __device__ inline Affine lcg_jump(uint64_t delta, uint64_t inc) {
    uint64_t acc_a = 1, acc_c = 0, cur_a = kPcgMult, cur_c = inc;
    while (delta) {
        if (delta & 1u) {
            acc_a *= cur_a;
            acc_c = acc_c * cur_a + cur_c;
        }
        cur_c = (cur_a + 1u) * cur_c;
        cur_a *= cur_a;
        delta >>= 1u;
    }
    return {acc_a, acc_c};
}

// pcg32_srandom_r(initstate = seed, initseq = stream_id), then skip `offset`.
struct StreamStart {
    uint64_t state;  // state whose output is sample `offset`
    uint64_t inc;
};
__host__ __device__ inline StreamStart pcg32_start(uint64_t seed, uint64_t stream_id, uint64_t offset) {
    const uint64_t inc = (stream_id << 1u) | 1u;
    uint64_t s = inc;  // 0 * M + inc
    s += seed;
    s = s * kPcgMult + inc;
    const Affine j = lcg_jump(offset, inc);
    return {j.a * s + j.c, inc};
}

// s' = a s + c (mod 2^64): IMAD.WIDE (low product + 64-bit addend), the two
// cross terms into the high word, and their sum.
__device__ __forceinline__ uint64_t lcg_step(uint64_t s, uint64_t a, uint64_t c) { return a * s + c; }

// Opaque copy: stops ptxas from folding a kernel-parameter constant into
// uniform registers (IMAD.WIDE cannot take a uniform 64-bit addend).
__device__ __forceinline__ uint64_t as_register(uint64_t x) {
    uint64_t r;
    asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(x));
    return r;
}

// Packed f32x2 (sm_100 FADD2 / FMUL2 / FFMA2), round-to-nearest per lane.
__device__ __forceinline__ uint64_t pack2(uint32_t lo, uint32_t hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}
// Float pair as one f32x2 register.  Written with float operands so that
// ptxas can fold per-half sign / abs modifiers into the consuming FADD2
// (-|x| costs nothing there, where an integer sign OR is a LOP3 per lane).
__device__ __forceinline__ uint64_t pack2f(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ uint32_t lo32(uint64_t x) { return static_cast<uint32_t>(x); }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return static_cast<uint32_t>(x >> 32); }

// One PCG32 LCG step s' = M s + inc.  The low product and the increment go
// through one IMAD.WIDE; the two cross products are then accumulated on top
// of its high word in place (2 IMAD): 3 instructions and a 2-IMAD dependency
// chain per step, where `M * s + inc` compiles to 3 IMAD + 1 add.  `mlo` is
// the multiplier's low word in a register (with the literal the compiler
// turns the widening multiply into a 64-bit one and ptxas adds a stray
// zero high word per step).
#ifndef ARV_LCG3
#define ARV_LCG3 1
#endif
__device__ __forceinline__ void lcg_step_pcg(uint32_t &lo, uint32_t &hi, uint64_t inc, uint32_t mlo) {
#if ARV_LCG3
    constexpr uint32_t mhi = static_cast<uint32_t>(kPcgMult >> 32);
    const uint64_t r = static_cast<uint64_t>(lo) * mlo + inc;
    uint32_t rl, h;  // inline PTX: written as C, the compiler re-associates the sum into 2 IMAD + IADD3
    asm("mov.b64 {%0, %1}, %2;" : "=r"(rl), "=r"(h) : "l"(r));
    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(hi), "r"(mlo));
    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(lo), "r"(mhi));
    lo = rl;
    hi = h;
#else
    const uint64_t s = lcg_step(pack2(lo, hi), kPcgMult, inc);
    lo = lo32(s);
    hi = hi32(s);
#endif
}
__device__ __forceinline__ uint64_t f32x2_add(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f32x2_mul(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f32x2_fma(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// a * b + c on the FMA pipe (IMAD), keeping the ALU pipe free.
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// ld.shared.f32 at a shared-space byte address plus an immediate offset.
template <int OFF>
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
    return v;
}

// ld.shared.v2.f32 (LDS.64) at a shared-space byte address.
__device__ __forceinline__ float2 lds_f32x2(uint32_t addr) {
    float2 v;
    asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

// XSH-RR output of a state (the value produced *before* stepping).
__device__ __forceinline__ uint32_t pcg32_output(uint64_t old) {
    const uint32_t lo = static_cast<uint32_t>(old);
    const uint32_t hi = static_cast<uint32_t>(old >> 32);
    // bits 27..58 of (old ^ (old >> 18)) = funnel(lo,hi,27) ^ (hi >> 13)
    const uint32_t xs = __funnelshift_r(lo, hi, 27) ^ (hi >> 13);
    const uint32_t rot = hi >> 27;
    return __funnelshift_r(xs, xs, rot);
}

#ifndef ARV_PCG_IMADHI
#define ARV_PCG_IMADHI 0
#endif
// Same output with the two right shifts of `hi` done as IMAD.HI (high word of
// hi * 2^k) on the FMA pipe, balancing the ALU-heavy XSH-RR.  m19 = 2^19,
// m5 = 2^5 must arrive in registers (not immediates), or ptxas folds the
// multiply back into a shift.
__device__ __forceinline__ uint32_t pcg32_output_fma(uint32_t lo, uint32_t hi, uint32_t m19, uint32_t m5) {
#if ARV_PCG_IMADHI >= 1
    const uint32_t rot = __umulhi(hi, m5);  // hi >> 27
#else
    const uint32_t rot = hi >> 27;
#endif
#if ARV_PCG_IMADHI >= 2
    const uint32_t xs = __funnelshift_r(lo, hi, 27) ^ __umulhi(hi, m19);  // hi >> 13
#else
    const uint32_t xs = __funnelshift_r(lo, hi, 27) ^ (hi >> 13);
#endif
    return __funnelshift_r(xs, xs, rot);
}

// ------------------------------------------------------- Philox-4x64-10 --
// The reference's own uniform source (numpy.random.Philox behind
// UniformStream, sampler.py:26-66): key = [seed, stream_id], word n of the
// stream = Philox(ctr = [n/4 + 1, carry, 0, 0], key)[n % 4] (numpy
// pre-increments the 256-bit counter), u = ((w >> 11) + 0.5) 2^-53.
struct Philox4 {
    uint64_t w[4];
};
__device__ __forceinline__ Philox4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0,
                                                 uint64_t k1) {
    constexpr uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    constexpr uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += W0;
            k1 += W1;
        }
        const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
        const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    return {{c0, c1, c2, c3}};
}
// Word `n` of UniformStream(seed, stream_id).
__device__ __forceinline__ uint64_t philox_word(uint64_t n, uint64_t seed, uint64_t sid) {
    const uint64_t b = (n >> 2) + 1;
    const Philox4 r = philox4x64_10(b, b == 0 ? 1u : 0u, 0, 0, seed, sid);
    const int lane = static_cast<int>(n & 3);
    return lane == 0 ? r.w[0] : lane == 1 ? r.w[1] : lane == 2 ? r.w[2] : r.w[3];
}
// sampler.py:62: ((w >> 11) + 0.5) * 2^-53, exact.
__device__ __forceinline__ double u64_to_f64(uint64_t w) {
    return __dmul_rn(__dadd_rn(static_cast<double>(w >> 11), 0.5), 0x1p-53);
}

// ------------------------------------------------------ uniform mappings --
// f32 lattice uniform u = ((w >> 9) + 0.5) 2^-23, returned in reflected form:
//   m  = all-ones iff u >= 1/2 (i.e. the reference predicate u < 0.5 is false)
//   v  = min(u, 1-u) = (k' + 0.5) 2^-23 computed exactly as
//        as_float(0x3F800000 | k') - (1 - 2^-24)   (Sterbenz; no I2F)
struct Reflected {
    float v;
    uint32_t m;
};
__device__ __forceinline__ Reflected reflect_u32(uint32_t w) {
    const uint32_t m = static_cast<uint32_t>(static_cast<int32_t>(w) >> 31);
    const uint32_t kp = (w ^ m) >> 9;
    const float v = __fsub_rn(__uint_as_float(0x3F800000u | kp), 0.99999994f);
    return {v, m};
}
__device__ __forceinline__ float u32_to_f32(uint32_t w) {
    return __fmul_rn(__uint2float_rn(w >> 9) + 0.5f, 0x1p-23f);
}
__device__ __forceinline__ double u32_to_f64(uint32_t w) {
    return __dmul_rn(__dadd_rn(static_cast<double>(w), 0.5), 0x1p-32);
}

// The same f64 uniform as D = 1 + u assembled from the word's bits (sign 0,
// exponent 0x3FF, mantissa w . 1 . 0...): exact, so D - 1 == u32_to_f64(w)
// bit for bit without the I2F and DMUL; the reference's u > 1/2 is w >= 2^31
// (both pinned by tests/test_oracle.py::test_f64_uniform_integer_domain).
__device__ __forceinline__ double one_plus_u32(uint32_t w) {
    return __hiloint2double(static_cast<int>(0x3FF00000u | (w >> 12)), static_cast<int>((w << 20) | 0x80000u));
}

// ------------------------------------------------------ AS 241 (PPND16) --
// exact_dist.py:30-62 coefficients (constant term first); evaluation order of
// exact_dist.py:65-126.  Coefficients live in constant memory: every lane of
// a warp reads the same word, so they are broadcast operands of DMUL/DADD.
#define ARV_AS241_A 3.3871328727963666080e0, 1.3314166789178437745e2, 1.9715909503065514427e3, \
    1.3731693765509461125e4, 4.5921953931549871457e4, 6.7265770927008700853e4,                 \
    3.3430575583588128105e4, 2.5090809287301226727e3
#define ARV_AS241_B 1.0, 4.2313330701600911252e1, 6.8718700749205790830e2,                  \
    5.3941960214247511077e3, 2.1213794301586595867e4, 3.9307895800092710610e4,               \
    2.8729085735721942674e4, 5.2264952788528545610e3
#define ARV_AS241_C 1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0, \
    3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,                 \
    2.27238449892691845833e-2, 7.74545014278341407640e-4
#define ARV_AS241_D 1.0, 2.05319162663775882187e0, 1.67638483018380384940e0,                   \
    6.89767334985100004550e-1, 1.48103976427480074590e-1, 1.51986665636164571966e-2,          \
    5.47593808499534494600e-4, 1.05075007164441684324e-9
#define ARV_AS241_E 6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0, \
    2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,               \
    2.71155556874348757815e-5, 2.01033439929228813265e-7
#define ARV_AS241_F 1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1,                 \
    1.48753612908506148525e-2, 7.86869131145613259100e-4, 1.84631831751005468180e-5,          \
    1.42151175831644588870e-7, 2.04426310338993978564e-15

static __constant__ double kAS241d[6][8] = {{ARV_AS241_A}, {ARV_AS241_B}, {ARV_AS241_C},
                                            {ARV_AS241_D}, {ARV_AS241_E}, {ARV_AS241_F}};
// Same coefficients rounded to f32 (the single-precision evaluation).
static __constant__ float kAS241f[6][8] = {{ARV_AS241_A}, {ARV_AS241_B}, {ARV_AS241_C},
                                           {ARV_AS241_D}, {ARV_AS241_E}, {ARV_AS241_F}};

// Per-lane coefficient rows for as241_f64 / as241_f32 in global memory,
// interleaved (A_i, B_i) for the central rational and (C_i, D_i) for the near
// tail, so one 16-byte (f64) or 8-byte (f32) read-only load feeds both Horner
// chains at step i.  A warp touches at most the two rows: L1-resident.
template <typename T>
struct alignas(2 * sizeof(T)) AS241Pairs {
    T v[32];
};
template <typename T>
constexpr AS241Pairs<T> as241_pairs() {
    constexpr double A[8] = {ARV_AS241_A}, B[8] = {ARV_AS241_B}, C[8] = {ARV_AS241_C}, D[8] = {ARV_AS241_D};
    AS241Pairs<T> p{};
    for (int i = 0; i < 8; ++i) {
        p.v[2 * i] = static_cast<T>(A[i]);
        p.v[2 * i + 1] = static_cast<T>(B[i]);
        p.v[16 + 2 * i] = static_cast<T>(C[i]);
        p.v[16 + 2 * i + 1] = static_cast<T>(D[i]);
    }
    return p;
}
static __device__ const AS241Pairs<double> kAS241pd = as241_pairs<double>();
static __device__ const AS241Pairs<float> kAS241pf = as241_pairs<float>();

// num(x) / den(x) of the lane's rational (central A/B or near-tail C/D),
// Horner with separately rounded multiply and add in the reference's order.
// rows: the 16 (A_i, B_i) / (C_i, D_i) pairs staged in shared memory by the
// caller (as241_stage_rows), or nullptr to read them through the read-only path.
__device__ __forceinline__ void as241_rational(double x, bool central, double &num, double &den,
                                               const double2 *rows = nullptr) {
    if (rows) {
        const double2 *cf = rows + (central ? 0 : 8);
        double2 c = cf[7];
        num = c.x;
        den = c.y;
#pragma unroll
        for (int i = 6; i >= 0; --i) {
            c = cf[i];
            num = __dadd_rn(__dmul_rn(num, x), c.x);
            den = __dadd_rn(__dmul_rn(den, x), c.y);
        }
        return;
    }
    const double2 *cf = reinterpret_cast<const double2 *>(kAS241pd.v) + (central ? 0 : 8);
    double2 c = __ldg(cf + 7);
    num = c.x;
    den = c.y;
#pragma unroll
    for (int i = 6; i >= 0; --i) {
        c = __ldg(cf + i);
        num = __dadd_rn(__dmul_rn(num, x), c.x);
        den = __dadd_rn(__dmul_rn(den, x), c.y);
    }
}
// Copy the AS241 coefficient pairs to shared memory (16 double2; the caller
// synchronises the CTA before use).
__device__ __forceinline__ void as241_stage_rows(double2 *rows) {
    if (threadIdx.x < 16) rows[threadIdx.x] = reinterpret_cast<const double2 *>(kAS241pd.v)[threadIdx.x];
}
__device__ __forceinline__ void as241_rational(float x, bool central, float &num, float &den) {
    const float2 *cf = reinterpret_cast<const float2 *>(kAS241pf.v) + (central ? 0 : 8);
    float2 c = __ldg(cf + 7);
    num = c.x;
    den = c.y;
#pragma unroll
    for (int i = 6; i >= 0; --i) {
        c = __ldg(cf + i);
        num = __fadd_rn(__fmul_rn(num, x), c.x);
        den = __fadd_rn(__fmul_rn(den, x), c.y);
    }
}

// Horner with separately rounded multiply and add (numpy has no FMA).
__device__ __forceinline__ double poly8d(int which, double x) {
    double acc = kAS241d[which][7];
#pragma unroll
    for (int i = 6; i >= 0; --i) acc = __dadd_rn(__dmul_rn(acc, x), kAS241d[which][i]);
    return acc;
}
__device__ __forceinline__ float poly8f(int which, float x) {
    float acc = kAS241f[which][7];
#pragma unroll
    for (int i = 6; i >= 0; --i) acc = __fadd_rn(__fmul_rn(acc, x), kAS241f[which][i]);
    return acc;
}

// Reference-order evaluation, one branch per region (kept for the rare far
// tail r > 5 and as the readable statement of exact_dist.py:87-126).
__device__ __forceinline__ double as241_f64_branchy(double u) {
    const double q = __dsub_rn(u, 0.5);
    if (fabs(q) <= 0.425) {
        const double r = __dsub_rn(0.180625, __dmul_rn(q, q));
        return __ddiv_rn(__dmul_rn(q, poly8d(0, r)), poly8d(1, r));
    }
    const bool upper = u > 0.5;
    const double w = upper ? __dsub_rn(1.0, u) : u;
    const double r = __dsqrt_rn(-log(w));
    double val;
    if (r <= 5.0) {
        const double rn = __dsub_rn(r, 1.6);
        val = __ddiv_rn(poly8d(2, rn), poly8d(3, rn));
    } else {
        const double rf = __dsub_rn(r, 5.0);
        val = __ddiv_rn(poly8d(4, rf), poly8d(5, rf));
    }
    return upper ? val : -val;
}

// Same results, fewer divergent FP64 instructions: a warp almost always holds
// both central and near-tail lanes (SURVEY §7 vi), so instead of executing
// both rational functions it evaluates ONE degree-7/7 rational whose
// coefficients are selected per lane (A/B central, C/D near tail) -- the
// selects run on the otherwise idle integer pipe, the Horner steps and the
// division keep the reference's operation order, so every lane is rounded
// exactly as in as241_f64_branchy.  Only the log/sqrt of the tail and the
// r > 5 far tail (u < ~1.4e-11) stay divergent.
// Core with the region predicates and q = u - 1/2 supplied by the caller
// (the PCG32 level kernels derive u > 1/2 from the word).
__device__ __forceinline__ double as241_f64_core(double u, double q, bool central, bool upper) {
    double x;
    if (central) {
        x = __dsub_rn(0.180625, __dmul_rn(q, q));
    } else {
        const double w = upper ? __dsub_rn(1.0, u) : u;
        const double r = __dsqrt_rn(-log(w));
        if (r > 5.0) return as241_f64_branchy(u);
        x = __dsub_rn(r, 1.6);
    }
    double num, den;
    as241_rational(x, central, num, den);
    const double val = __ddiv_rn(central ? __dmul_rn(q, num) : num, den);
    return central || upper ? val : -val;
}

__device__ __forceinline__ double as241_f64(double u) {
    const double q = __dsub_rn(u, 0.5);
    return as241_f64_core(u, q, fabs(q) <= 0.425, u > 0.5);
}

// N evaluations per lane with the tail's log / sqrt compacted across the warp.
// A warp of independent lanes almost always holds some tail value (|u - 1/2|
// > 0.425 has probability 0.15; P(no tail among 32 lanes) = 0.5%), so
// per-element calls run the ~100-instruction log + sqrt once per element for
// the whole warp.  Here the warp's pending tails are compacted through a
// per-warp shared-memory list and served 32 at a time: one log + sqrt pass per
// 32 tails of the warp (0.6 per 4 uniforms on average, so one pass for
// nearly every N = 4 batch).  The earlier per-lane form (ARV_AS241_SMEM_COMPACT
// = 0) served the lowest pending tail of every lane per pass: as many passes
// as the busiest lane has tails (about 1.5 for N = 2 and 2.3 for N = 4).
// Every element still goes through exactly the operations of
// as241_f64_core, so results are identical.
// LIST selects the shared-memory list (GBM level kernels: 19.9 -> 17.6 ms for
// config 4); the standalone AS241 kernels keep the per-lane passes, which
// measured 2% faster there (0.996 vs 1.014 ms for gauss64).
#ifndef ARV_AS241_SMEM_COMPACT
#define ARV_AS241_SMEM_COMPACT 1
#endif
constexpr int kTailWarps = 8;  // callers launch <= 256 threads per CTA
template <int N, bool LIST = false>
__device__ __forceinline__ void as241_f64_batch(const double (&u)[N], double (&out)[N],
                                                const double2 *rows = nullptr) {
    double q[N], x[N];
    unsigned pend = 0, central = 0, upper = 0, far = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        q[k] = __dsub_rn(u[k], 0.5);
        if (fabs(q[k]) <= 0.425) central |= 1u << k;
        else pend |= 1u << k;
        if (u[k] > 0.5) upper |= 1u << k;
        x[k] = __dsub_rn(0.180625, __dmul_rn(q[k], q[k]));  // central argument; tails overwrite it
    }
    const unsigned am = __activemask();
    if constexpr (LIST && ARV_AS241_SMEM_COMPACT) {
    // Every pending tail of the warp goes to a per-warp shared-memory list;
    // the active lanes take its entries round-robin (one log + sqrt per
    // 32 tails instead of one per busiest lane's tail) and the results return
    // through the same slots.  Same operations per element.
    static_assert(N <= 4, "tail buffer holds 4 elements per lane");
    __shared__ double tail_buf[kTailWarps][32 * 4];
    double *buf = tail_buf[threadIdx.x >> 5];
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    int pos[N];
    int total = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const unsigned b = __ballot_sync(am, (pend >> k) & 1u);
        pos[k] = total + __popc(b & lt);
        total += __popc(b);
    }
    if (total) {  // warp-uniform
#pragma unroll
        for (int k = 0; k < N; ++k)
            if ((pend >> k) & 1u) buf[pos[k]] = (upper >> k) & 1u ? __dsub_rn(1.0, u[k]) : u[k];
        __syncwarp(am);
        const int na = __popc(am);
        for (int g = __popc(am & lt); g < total; g += na) buf[g] = __dsqrt_rn(-log(buf[g]));
        __syncwarp(am);
#pragma unroll
        for (int k = 0; k < N; ++k)
            if ((pend >> k) & 1u) {
                const double r = buf[pos[k]];
                x[k] = __dsub_rn(r, 1.6);
                if (r > 5.0) far |= 1u << k;
            }
        __syncwarp(am);  // the list is reused by the next call
    }
    } else {
    while (__any_sync(am, pend != 0u)) {
        // Lanes without a pending tail evaluate a dummy log(1/2): with w = 1 the
        // sqrt argument would be -0, which sends the whole warp through
        // __dsqrt_rn's out-of-range slow path on every pass.
        double w = 0.5;
        int sel = -1;
#pragma unroll
        for (int k = N - 1; k >= 0; --k)
            if (pend & (1u << k)) {
                sel = k;
                w = (upper >> k) & 1u ? __dsub_rn(1.0, u[k]) : u[k];
            }
        const double r = __dsqrt_rn(-log(w));
#pragma unroll
        for (int k = 0; k < N; ++k)
            if (k == sel) {
                x[k] = __dsub_rn(r, 1.6);
                if (r > 5.0) far |= 1u << k;
            }
        pend &= pend - 1u;
    }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const bool c = (central >> k) & 1u;
        double num, den;
        as241_rational(x[k], c, num, den, rows);
        const double val = __ddiv_rn(c ? __dmul_rn(q[k], num) : num, den);
        out[k] = c || ((upper >> k) & 1u) ? val : -val;
    }
    if (far) {  // r > 5 (u < ~1.4e-11 or > 1 - 1.4e-11): E/F rational, rare
#pragma unroll
        for (int k = 0; k < N; ++k)
            if ((far >> k) & 1u) out[k] = as241_f64_branchy(u[k]);
    }
}

__device__ __forceinline__ float as241_f32_branchy(float u) {
    const float q = __fsub_rn(u, 0.5f);
    if (fabsf(q) <= 0.425f) {
        const float r = __fsub_rn(0.180625f, __fmul_rn(q, q));
        return __fdiv_rn(__fmul_rn(q, poly8f(0, r)), poly8f(1, r));
    }
    const bool upper = u > 0.5f;
    const float w = upper ? __fsub_rn(1.0f, u) : u;
    const float r = __fsqrt_rn(-logf(w));
    float val;
    if (r <= 5.0f) {
        const float rn = __fsub_rn(r, 1.6f);
        val = __fdiv_rn(poly8f(2, rn), poly8f(3, rn));
    } else {
        const float rf = __fsub_rn(r, 5.0f);
        val = __fdiv_rn(poly8f(4, rf), poly8f(5, rf));
    }
    return upper ? val : -val;
}

// Same results as as241_f32_branchy with one rational per lane (see as241_f64).
__device__ __forceinline__ float as241_f32(float u) {
    const float q = __fsub_rn(u, 0.5f);
    const bool central = fabsf(q) <= 0.425f;
    const bool upper = u > 0.5f;
    float x;
    if (central) {
        x = __fsub_rn(0.180625f, __fmul_rn(q, q));
    } else {
        const float w = upper ? __fsub_rn(1.0f, u) : u;
        const float r = __fsqrt_rn(-logf(w));
        if (r > 5.0f) return as241_f32_branchy(u);
        x = __fsub_rn(r, 1.6f);
    }
    float num, den;
    as241_rational(x, central, num, den);
    const float val = __fdiv_rn(central ? __fmul_rn(q, num) : num, den);
    return central || upper ? val : -val;
}

// ------------------------------------------------- dyadic index helpers --
// _kernels.pyx:36 / :51 (exponent bits), capped at `cap` like the reference.
// There is no lower clamp here: u > 1/2 or u = 1 gives a negative index
// (dyadic_index32(1.0) = -1 in the reference), so callers that index a table
// with the result clamp it at 0 themselves.
__device__ __forceinline__ long long dyadic_idx64(double v, long long cap) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    const long long idx = 1022 - static_cast<long long>(bits >> 52);
    return idx < cap ? idx : cap;
}
__device__ __forceinline__ long long dyadic_idx32(float v, long long cap) {
    const unsigned int bits = __float_as_uint(v);
    const long long idx = 126 - static_cast<long long>(bits >> 23);
    return idx < cap ? idx : cap;
}

// Grid for a streaming kernel: enough CTAs to fill every SM `per_sm` times,
// never more than the work needs.
inline int stream_grid(int64_t work_items, int block, int per_sm) {
    const int64_t need = (work_items + block - 1) / block;
    const int64_t cap = static_cast<int64_t>(device_sm_count()) * per_sm;
    int64_t g = need < cap ? need : cap;
    return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace arv

// Fused PCG32 -> inverse-CDF generators.
//
// One thread owns a PCG32 state in registers and produces groups of G = 4 or
// 8 consecutive samples (G*g .. G*g+G-1 for its group index g), written with
// one st.global.v4 (128-bit) or st.global.v8 (256-bit, sm_100) per group, so
// every warp store is fully coalesced and the only HBM traffic is the output.
// Within a group the LCG steps once per sample; between groups the thread
// jumps over the G(T-1) samples the other T-1 threads own with one affine
// map (A, C) = LCG^(G T - G + 1), precomputed on the host.  Output i of a
// call is PCG32 output (offset + i) of stream (seed, stream_id) whatever the
// grid or G, so shards on different GPUs concatenate bit-exactly.
//
// Evaluators (reference semantics, see oracle/oracle.c):
//   constant   values[floor(2^q u)]            (_kernels.pyx:16-23)
//   subdyadic  octave x sub-interval Horner    (_kernels.pyx:76-93 when sub_bits = 0)
//   uniform    u itself; gaussian32/64 = AS241 (exact_dist.py:87-126)
#include <algorithm>

#include "arv_common.cuh"

namespace arv {

// ------------------------------------------------------------ tuning ----
// Compile-time variants (tools/prof_kernels.py builds them for sweeps):
//   ARV_GEN_MINB    min resident CTAs per SM for __launch_bounds__ (register cap)
//   ARV_GEN_UNROLL  groups per loop iteration
// Sweep (B200, 2^28 samples, r01): MINB 6 / UNROLL 2 / group 8 / 8 CTAs per
// SM was fastest for the sub-interval generator (0.206 ms vs 0.224-0.243 ms
// for the other variants, incl. split half-chains).
#ifndef ARV_GEN_MINB
#define ARV_GEN_MINB 6
#endif
#ifndef ARV_GEN_PDL
#define ARV_GEN_PDL 1
#endif
#ifndef ARV_GEN_UNROLL
#define ARV_GEN_UNROLL 2
#endif
constexpr int kGenUnroll = ARV_GEN_UNROLL;
#ifndef ARV_SIGNED_UNROLL
#define ARV_SIGNED_UNROLL 1
#endif
constexpr int kSignedUnroll = ARV_SIGNED_UNROLL;  // the signed-table generator (headline)
// Process-wide launch shape knobs (arv_set_tuning); defaults from sweeps.
static int g_group = 8;        // samples per thread-group: 4 (v4) or 8 (v8)
static int g_ctas_per_sm = 0;  // CTAs per SM (256 threads each); 0 = auto (see gen_grid)
// calls of at least this many samples take the lane-table kernel (< 0: never).  Back to back
// (tools/lane_threshold.py) it ties with the signed-table kernel at 2^22-2^23, loses 1-6% at
// 2^24-2^25 (57 KB staged per CTA) and wins from 2^26 on (2^28: 3.6%).
static int64_t g_lane_min_n = int64_t{1} << 26;
extern int g_cir_segment;      // arv_mlmc.cu
extern int g_gbm_kernel;       // arv_mlmc.cu
int set_nc_certify(int on);    // arv_mlmc.cu

constexpr int kJumpBits = 24;  // grid threads < 2^24

struct GenArgs {
    uint64_t s_base;  // state whose output is sample 0 of this call
    uint64_t inc;
    Affine stride;    // LCG^(G T - G + 1)
    int64_t n;
    uint64_t zero;    // always 0: makes derived constants per-thread registers
    uint32_t zero32;
    uint64_t iter_q, iter_r;  // (n / G) = iter_q * T + iter_r: thread g0 runs iter_q + (g0 < iter_r) groups
    Affine pow2[kJumpBits];  // LCG^(G 2^i): a thread reaches group g0 with popcount(g0) steps
};

// State of the first sample of group g0 = blockIdx.x * 256 + threadIdx.x
// (g0 < 2^kJumpBits, blockDim.x = 256): thread 0 walks the CTA's high bits
// once and shares the state; each thread then walks only its 8 low bits
// (powers of one affine map commute).  A full 24-bit walk per thread was ~20%
// of a thread's work at 2^24 samples.
template <int LB>  // log2(blockDim.x); s_cta: a shared-memory slot for the CTA's state
__device__ __forceinline__ uint64_t group_start(const GenArgs &a, uint64_t g0, uint64_t &s_cta) {
    if (threadIdx.x == 0) {
        uint64_t s = a.s_base;
        const uint64_t hb = g0 >> LB;
#pragma unroll 1
        for (int i = LB; i < kJumpBits && (hb >> (i - LB)) != 0; ++i)
            if ((g0 >> i) & 1u) s = a.pow2[i].a * s + a.pow2[i].c;
        s_cta = s;
    }
    __syncthreads();
    uint64_t s = s_cta;
#pragma unroll
    for (int i = 0; i < LB; ++i)
        if ((g0 >> i) & 1u) s = a.pow2[i].a * s + a.pow2[i].c;
    return s;
}
template <int LB = 8>
__device__ __forceinline__ uint64_t group_start(const GenArgs &a, uint64_t g0) {
    __shared__ uint64_t s_cta;
    return group_start<LB>(a, g0, s_cta);
}

static GenArgs make_gen_args(uint64_t seed, uint64_t stream_id, uint64_t offset, int64_t n,
                             int64_t total_threads, int G) {
    const StreamStart st = pcg32_start(seed, stream_id, offset);
    GenArgs a;
    a.s_base = st.state;
    a.inc = st.inc;
    a.stride = lcg_jump(static_cast<uint64_t>(G) * static_cast<uint64_t>(total_threads) - (G - 1), st.inc);
    a.n = n;
    a.zero = 0;
    a.zero32 = 0;
    const uint64_t n_full = static_cast<uint64_t>(n) / static_cast<uint64_t>(G);
    a.iter_q = n_full / static_cast<uint64_t>(total_threads);
    a.iter_r = n_full % static_cast<uint64_t>(total_threads);
    Affine p = lcg_jump(static_cast<uint64_t>(G), st.inc);
    for (int i = 0; i < kJumpBits; ++i) {
        a.pow2[i] = p;
        p = {p.a * p.a, p.a * p.c + p.c};  // compose the map with itself
    }
    return a;
}

template <int G>
struct VecOut;
template <>
struct VecOut<4> {
    __device__ __forceinline__ static void store(uint32_t *p, const uint32_t (&r)[4]) {
        __stcs(reinterpret_cast<uint4 *>(p), make_uint4(r[0], r[1], r[2], r[3]));
    }
};
template <>
struct VecOut<8> {
    __device__ __forceinline__ static void store(uint32_t *p, const uint32_t (&r)[8]) {
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]),
                     "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                     : "memory");
    }
};

// Evaluate two samples: the evaluator's packed-pair path when it has one.
template <class Eval, class = void>
struct HasPair {
    static constexpr bool value = false;
};
template <class Eval>
struct HasPair<Eval, decltype(void(Eval::kHasPair))> {
    static constexpr bool value = Eval::kHasPair;
};
template <class Eval>
__device__ __forceinline__ void eval_two(const Eval &eval, uint32_t w0, uint32_t w1, uint32_t &r0, uint32_t &r1) {
    if constexpr (HasPair<Eval>::value) {
        eval.pair(w0, w1, r0, r1);
    } else {
        r0 = eval(w0);
        r1 = eval(w1);
    }
}

// The group loop: thread g0 starts at state `s` (its first group) and
// produces its groups with G-wide stores (out must be 4*G-byte aligned).
template <int G, int U = kGenUnroll, class Eval>
__device__ __forceinline__ void gen_run(const GenArgs &a, uint32_t *__restrict__ out, const Eval &eval, uint64_t s,
                                        uint64_t g0) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t n_full = static_cast<uint64_t>(a.n) / G;
    const uint64_t z = static_cast<uint64_t>(threadIdx.x) * a.zero;  // 0, but not provably uniform
    const uint64_t inc = a.inc + z;
    const Affine st{a.stride.a + z, a.stride.c + z};
    const uint32_t mlo = static_cast<uint32_t>(kPcgMult) + static_cast<uint32_t>(z);
    const uint32_t m19 = (1u << 19) + static_cast<uint32_t>(z), m5 = 32u + static_cast<uint32_t>(z);
    // Trip count once; the loop runs on a 32-bit counter and a pointer bump.
    // host-computed quotient / remainder: no 64-bit division per thread
    const uint32_t iters = static_cast<uint32_t>(a.iter_q) + (g0 < a.iter_r ? 1u : 0u);
    uint32_t *p = out + G * g0;
    const uint64_t step = G * T;
#pragma unroll U
    for (uint32_t it = 0; it < iters; ++it) {
        uint32_t w[G];
        uint32_t slo, shi;  // the state as two words: the low product is then one widening multiply
        asm("mov.b64 {%0, %1}, %2;" : "=r"(slo), "=r"(shi) : "l"(s));
#pragma unroll
        for (int i = 0; i < G; ++i) {
            w[i] = pcg32_output_fma(slo, shi, m19, m5);
            if (i < G - 1) lcg_step_pcg(slo, shi, inc, mlo);
        }
        s = lcg_step(pack2(slo, shi), st.a, st.c);
        uint32_t r[G];
#pragma unroll
        for (int i = 0; i < G; i += 2) eval_two(eval, w[i], w[i + 1], r[i], r[i + 1]);
        VecOut<G>::store(p, r);
        p += step;
    }
    const uint64_t g = g0 + static_cast<uint64_t>(iters) * T;
    const int rem = static_cast<int>(a.n % G);
    if (g == n_full && rem) {
        for (int i = 0; i < rem; ++i) {
            out[G * g + i] = eval(pcg32_output(s));
            s = lcg_step(s, kPcgMult, inc);
        }
    }
}

__device__ __forceinline__ void pdl_wait() {
#if ARV_GEN_PDL
    // Programmatic dependent launch: everything before this may overlap the
    // previous kernel's tail on the stream; wait for it to complete (and its
    // stores to be visible) before reading a table or storing.
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// Drive `eval(w) -> uint32 bits` over the call's samples with G-wide stores.
// `stage()` runs after griddepcontrol.wait and before the first store: it
// stages the kernel's table into shared memory, so a table written by the
// previous kernel on the stream is visible (PDL RAW ordering).  Only the
// parameter-only start-state walk overlaps the predecessor's tail.
template <int G, class Eval, class Stage>
__device__ __forceinline__ void gen_loop_vec(const GenArgs &a, uint32_t *__restrict__ out, const Eval &eval,
                                             const Stage &stage) {
    const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t s = group_start<>(a, g0);
    pdl_wait();
    stage();
    gen_run<G>(a, out, eval, s, g0);
}

// Scalar-store variant for outputs that are not 16-byte aligned.
template <class Eval, class Stage>
__device__ __forceinline__ void gen_loop_v1(uint64_t s_base, uint64_t inc, int64_t n, uint32_t *__restrict__ out,
                                            const Eval &eval, const Stage &stage) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Affine j0 = lcg_jump(i, inc);
    const Affine sT = lcg_jump(T, inc);
    uint64_t s = j0.a * s_base + j0.c;
#if ARV_GEN_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    stage();
    for (; i < static_cast<uint64_t>(n); i += T) {
        out[i] = eval(pcg32_output(s));
        s = lcg_step(s, sT.a, sT.c);
    }
}

// MODE: 1 = scalar stores (unaligned out), 4 = v4, 8 = v8.
struct NoStage {
    __device__ __forceinline__ void operator()() const {}
};
template <int MODE, class Eval, class Stage = NoStage>
__device__ __forceinline__ void gen_dispatch(const GenArgs &a, uint32_t *out, const Eval &ev,
                                             const Stage &stage = Stage{}) {
    if constexpr (MODE == 1) gen_loop_v1(a.s_base, a.inc, a.n, out, ev, stage);
    else gen_loop_vec<MODE>(a, out, ev, stage);
}

// ------------------------------------------------------------ evaluators --
struct EvalWord {
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const { return w; }
};
struct EvalUniform {
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        return __float_as_uint(u32_to_f32(w));
    }
};
struct EvalGauss32 {
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        return __float_as_uint(as241_f32(u32_to_f32(w)));
    }
};
// floor(2^q u) for u = (k + 1/2) 2^-23, k = w >> 9: k >> (23-q) for q <= 23,
// 2k + 1 for q = 24.  Table in shared memory (q <= 14, addressed as a 32-bit
// shared-space address so the lookup is one LDS -- a generic pointer made it a
// generic LD with 64-bit address arithmetic) or global (L2).
struct EvalConstantSmem {
    uint32_t base;  // shared-space byte address of the table
    int shift;      // 32 - q
    uint32_t four;  // 4 in a register: the address is one IMAD
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        return __float_as_uint(lds_f32<0>(mad_u32(w >> shift, four, base)));
    }
};
struct EvalConstantGlobal {
    const float *tab;
    int shift;  // 32 - q
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const { return __float_as_uint(__ldg(tab + (w >> shift))); }
};
struct EvalConstant24 {
    const float *tab;
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        return __float_as_uint(__ldg(tab + ((((w >> 9) << 1) | 1u))));
    }
};

// Octave x sub-interval on the f32 lattice.  v = min(u, 1-u) is built
// exactly in the FP pipe:  f = as_float(0x3F000000 | (w >> 9)) = 1/2 + t 2^-24,
// d = 2 (f - 3/4) + 2^-24 = u - 1/2 (exact, never 0), v = 1/2 - |d|.  The
// sign of d is the reference predicate (u < 1/2 <=> d < 0).  On the lattice
// v lies in [2^-24, 1/2), so its biased exponent E is 103..125 and
// bits(v) >> (23 - b) = (E << b) | sub indexes a "lattice table" of
// 23 << b entries per coefficient plane directly (the base offset 103 << b
// is folded into the shared-memory base address); octaves j = 126 - E >= K
// hold the singular polynomial.  Planes are separate f32 arrays at a fixed
// stride (one address IMAD, immediate offsets), so the four most frequent
// octaves (94% of samples) hit disjoint banks.
constexpr int kLatticeE0 = 103;                   // exponent of 2^-24
constexpr int kLatticeOct = 23;                   // octaves 1..23 on the f32 lattice
constexpr int kLatticePlane = kLatticeOct << 5;   // plane stride (max sub_bits = 5)

template <int DEG>
struct EvalSubDyadic {
    uint32_t base;  // shared-space byte address of plane 0, pre-offset by -4 (103 << b)
    int shift;
    uint32_t four;  // 4, held in a register so the address is one IMAD (FMA pipe)
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        const float f = __uint_as_float(0x3F800000u | (w >> 9));        // 1 + u - 2^-24, in [1, 2)
        const float d = __fadd_rn(__fadd_rn(f, -1.5f), 0x1p-24f);       // u - 1/2, exact
        const float v = __fadd_rn(0.5f, -fabsf(d));                     // 1/2 - |u - 1/2|, exact
        const uint32_t addr = mad_u32(__float_as_uint(v) >> shift, four, base);
        float z = lds_f32<DEG * kLatticePlane * 4>(addr);
#pragma unroll
        for (int k = DEG - 1; k >= 0; --k) {
            float c;
            switch (k) {  // immediate plane offsets
                case 0: c = lds_f32<0>(addr); break;
                case 1: c = lds_f32<1 * kLatticePlane * 4>(addr); break;
                case 2: c = lds_f32<2 * kLatticePlane * 4>(addr); break;
                case 3: c = lds_f32<3 * kLatticePlane * 4>(addr); break;
                default: c = lds_f32<4 * kLatticePlane * 4>(addr); break;
            }
            z = __fadd_rn(__fmul_rn(z, v), c);  // separately rounded (no FMA): reference parity
        }
        return __float_as_uint(z) ^ (~__float_as_uint(d) & 0x80000000u);
    }

    // Two samples at once with sm_100's packed f32x2 FP instructions
    // (FADD2 / FFMA2 / FMUL2: one issue slot for both lanes of the pair).
    // Each lane is rounded exactly as the scalar path (IEEE rn, the product
    // and the sum still separately rounded), so results are bit-identical.
    static constexpr bool kHasPair = DEG == 1;
    __device__ __forceinline__ void pair(uint32_t w0, uint32_t w1, uint32_t &r0, uint32_t &r1) const {
        // f = 1 + u - 2^-24 from the word's bits; d = (f - 3/2) + 2^-24 = u - 1/2
        // and v = 1/2 - |d| are exact: three FADD2 with immediate operands,
        // the -|d| folded into the last one as an operand modifier.
        const uint64_t f = pack2(0x3F800000u | (w0 >> 9), 0x3F800000u | (w1 >> 9));
        const uint64_t d = f32x2_add(f32x2_add(f, kMinus15x2), kUlp24x2);
        const uint32_t d0 = lo32(d), d1 = hi32(d);
        const uint64_t v = f32x2_add(kHalf2, pack2f(-fabsf(__uint_as_float(d0)), -fabsf(__uint_as_float(d1))));
        const uint32_t a0 = mad_u32(lo32(v) >> shift, four, base);
        const uint32_t a1 = mad_u32(hi32(v) >> shift, four, base);
        const uint64_t c1 = pack2(__float_as_uint(lds_f32<kLatticePlane * 4>(a0)),
                                  __float_as_uint(lds_f32<kLatticePlane * 4>(a1)));
        const uint64_t c0 = pack2(__float_as_uint(lds_f32<0>(a0)), __float_as_uint(lds_f32<0>(a1)));  // scalar use
        // Product packed, sum scalar: ptxas contracts mul.rn.f32x2 + add.rn.f32x2
        // into FFMA2 (one rounding), which would break parity with the
        // reference's separately rounded z*v + c; FMUL2 + 2 FADD stays exact.
        const uint64_t p = f32x2_mul(c1, v);
        const float z0 = __fadd_rn(__uint_as_float(lo32(p)), __uint_as_float(lo32(c0)));
        const float z1 = __fadd_rn(__uint_as_float(hi32(p)), __uint_as_float(hi32(c0)));
        r0 = __float_as_uint(z0) ^ (~d0 & 0x80000000u);
        r1 = __float_as_uint(z1) ^ (~d1 & 0x80000000u);
    }
    static constexpr uint64_t kMinus15x2 = 0xBFC00000BFC00000ull;   // {-1.5, -1.5}
    static constexpr uint64_t kUlp24x2 = 0x3380000033800000ull;     // {2^-24, 2^-24}
    static constexpr uint64_t kHalf2 = 0x3F0000003F000000ull;       // {0.5, 0.5}
};

// Stage natural-layout coeffs (DEG+1, K, nsub) into the lattice table.
template <int DEG>
__device__ __forceinline__ void stage_subdyadic(float *sm, const float *__restrict__ coeffs, int K, int b) {
    const int nsub = 1 << b;
    const int plane = kLatticeOct << b;
    for (int e = threadIdx.x; e < plane; e += blockDim.x) {
        const int E = kLatticeE0 + (e >> b), s = e & (nsub - 1);
        const int j = 126 - E;  // octave 1..23
        const int jj = j < K ? j : K;
        const int ss = j < K ? s : 0;
        for (int d = 0; d <= DEG; ++d)
            sm[d * kLatticePlane + e] = __ldg(coeffs + (static_cast<int64_t>(d) * K + (jj - 1)) * nsub + ss);
    }
    __syncthreads();
}

// Degree-1 octave x sub-interval evaluator with the reflection's sign folded
// into the table ("signed lattice table"), bit-identical to EvalSubDyadic<1>.
//   i  = (int32)w >> 9 (the lattice index k = w >> 9 less 2^23 when u >= 1/2),
//   g  = as_float(0x4B400000 + i) = 12582912 + i   (one LEA.HI.SX32),
//   vh = (g - 12582912) + 1/2 = i + 1/2            (two exact FADD2 per pair).
// For u < 1/2, vh = u 2^23 > 0; for u >= 1/2, vh = (u - 1) 2^23 = -(1 - u) 2^23,
// so |vh| = v 2^23 with v = min(u, 1 - u) and sign(vh) is the reference's
// predicate.  The table is indexed by bits(vh) >> (23 - b) = s|E|sub: entry
// (c0, c1 2^-23) for vh > 0 and (-c0, c1 2^-23) for vh < 0, so
//   RN(RN(c1' vh) + c0') = RN(c0 + RN(c1 v))  (vh > 0)
//                        = -RN(c0 + RN(c1 v)) (vh < 0; RN is odd-symmetric)
// exactly the reference's separately rounded z = c1 v + c0 and its sign flip,
// with no reflection, no sign fix-up and one LDS.64 per sample.  Two
// conditions make it exact, both checked per table entry while staging
// (stage_linsigned): c1 2^-23 is exact (no subnormal rounding), and no lattice
// point of the entry gives z == 0 (the reference returns -0.0 there, the
// signed table +0.0).  If either fails the kernel runs EvalSubDyadic<1>.
constexpr int kSignedE0 = 126;  // exponent of |vh| = 1/2 (octave 23)

struct EvalLinSigned {
    uint32_t base;   // shared byte address of the float2 table, pre-offset by -8 (126 << b)
    int shift;       // 23 - b
    uint32_t eight;  // 8 in a register: the address is one IMAD
    __device__ __forceinline__ static uint32_t magic(uint32_t w) {
        return 0x4B400000u + static_cast<uint32_t>(static_cast<int32_t>(w) >> 9);  // LEA.HI.SX32
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        const float vh = __fadd_rn(__fadd_rn(__uint_as_float(magic(w)), -12582912.0f), 0.5f);
        const float2 c = lds_f32x2(mad_u32(__float_as_uint(vh) >> shift, eight, base));
        return __float_as_uint(__fadd_rn(__fmul_rn(c.y, vh), c.x));
    }
    static constexpr bool kHasPair = true;
    __device__ __forceinline__ void pair(uint32_t w0, uint32_t w1, uint32_t &r0, uint32_t &r1) const {
        const uint64_t g = pack2(magic(w0), magic(w1));
        const uint64_t vh = f32x2_add(f32x2_add(g, kMinusMagic2), kHalf2);
        const float2 c0 = lds_f32x2(mad_u32(lo32(vh) >> shift, eight, base));
        const float2 c1 = lds_f32x2(mad_u32(hi32(vh) >> shift, eight, base));
        r0 = __float_as_uint(__fadd_rn(__fmul_rn(c0.y, __uint_as_float(lo32(vh))), c0.x));
        r1 = __float_as_uint(__fadd_rn(__fmul_rn(c1.y, __uint_as_float(hi32(vh))), c1.x));
    }
    static constexpr uint64_t kMinusMagic2 = 0xCB400000CB400000ull;  // {-12582912, -12582912}
    static constexpr uint64_t kHalf2 = 0x3F0000003F000000ull;        // {0.5, 0.5}
};

// Shared bytes of the signed table for sub_bits b: entries [0, 23 << b) for
// vh > 0 and the same at +2^(8+b) for vh < 0 (bit 31 of bits(vh)).
__host__ __device__ constexpr int linsigned_entries(int b) { return (1 << (8 + b)) + (23 << b); }

// z = RN(RN(c1 v) + c0) in f32 at lattice point v = (m + 1/2) 2^-23.
__device__ __forceinline__ float lin_at(float c0, float c1, int64_t m) {
    const float v = __fmul_rn(static_cast<float>(m) + 0.5f, 0x1p-23f);  // exact (m < 2^22)
    return __fadd_rn(__fmul_rn(c1, v), c0);
}

// Entry e = (E - kSignedE0) << b | sub of the signed tables: its coefficients
// (c0, c1) from the natural-layout coeffs (2, K, 2^b), and whether the signed
// evaluation is bit-exact on it (c1 times the power of two `c1_scale` is
// exact, and no lattice point |vh| = m + 1/2 of the entry gives z == 0).
__device__ __forceinline__ bool linsigned_entry(const float *__restrict__ coeffs, int K, int b, int e, float c1_scale,
                                                float &c0, float &c1s) {
    const int nsub = 1 << b;
    const int E = kSignedE0 + (e >> b), sub = e & (nsub - 1);
    const int j = 149 - E;  // octave 1..23
    const int jj = j < K ? j : K;
    const int ss = j < K ? sub : 0;
    c0 = __ldg(coeffs + static_cast<int64_t>(jj - 1) * nsub + ss);
    const float c1 = __ldg(coeffs + (static_cast<int64_t>(K) + jj - 1) * nsub + ss);
    c1s = __fmul_rn(c1, c1_scale);
    bool ok = isfinite(c0) && isfinite(c1) && __fmul_rn(c1s, 1.0f / c1_scale) == c1;
    // lattice points |vh| = m + 1/2 inside [lo, hi) of this entry
    const float lo = __uint_as_float(static_cast<uint32_t>(E) << 23 | static_cast<uint32_t>(sub) << (23 - b));
    const float hi = __uint_as_float((static_cast<uint32_t>(E) << 23) + (static_cast<uint32_t>(sub + 1) << (23 - b)));
    const int64_t m_lo = static_cast<int64_t>(ceilf(lo - 0.5f));
    const int64_t m_hi = static_cast<int64_t>(ceilf(hi - 0.5f)) - 1;
    if (m_lo <= m_hi) {
        // z is monotone in m over the entry (v exact and increasing, RN
        // monotone), so its exact zeros form one contiguous run.  Ends of
        // one sign: no zero.  A sign change (the fit crosses 0 near
        // v = 1/2): bisect with strict signs at both ends -- a run of
        // zeros between them is always hit by some midpoint.
        const float za = lin_at(c0, c1, m_lo), zb = lin_at(c0, c1, m_hi);
        if (za == 0.0f || zb == 0.0f || !(isfinite(za) && isfinite(zb))) {
            ok = false;
        } else if ((za > 0.0f) != (zb > 0.0f)) {
            int64_t lo_m = m_lo, hi_m = m_hi;
            while (hi_m - lo_m > 1) {
                const int64_t mid = lo_m + (hi_m - lo_m) / 2;
                const float zm = lin_at(c0, c1, mid);
                if (zm == 0.0f) {
                    ok = false;
                    break;
                }
                if ((zm > 0.0f) == (za > 0.0f)) lo_m = mid;
                else hi_m = mid;
            }
        }
    }
    return ok;
}

// Stage natural-layout coeffs (2, K, 2^b) into the signed table; returns the
// CTA-wide verdict that the signed evaluation is bit-exact for this table.
__device__ __forceinline__ bool stage_linsigned(float2 *sm, const float *__restrict__ coeffs, int K, int b) {
    const int neg = 1 << (8 + b);
    bool ok = true;
    for (int e = threadIdx.x; e < (23 << b); e += blockDim.x) {
        float c0, c1s;
        ok &= linsigned_entry(coeffs, K, b, e, 0x1p-23f, c0, c1s);
        sm[e] = make_float2(c0, c1s);
        sm[neg + e] = make_float2(-c0, c1s);
    }
    return __syncthreads_and(ok) != 0;
}

// The signed table with lane-private copies ("lane table"): the headline
// kernel's shared-memory lookups without bank conflicts.  On the signed table
// above a warp's 32 random LDS.64 take 5.1 wavefronts of the SM's shared-memory
// data path (ncu: l1tex data-pipe 93% busy -- the kernel's actual limiter,
// not HBM and not instruction issue); here they take the minimum of 2.
//   vh = (i + 1/2) 2^-13 (same construction with the magic scaled by 2^-13),
//   so |vh| in [2^-14, 2^9) is a normal f16 and  h = cvt.rz.f16(vh)  is
//   s | E5 | m10 with E5 = 1..23 (octave 24 - E5) and the top mantissa bits
//   the sub-interval (truncation: the index never rounds up).
// Row r = h >> (10 - b) starts at byte (h & mask), mask = 0xFFFF << (10 - b):
// for b <= 3 a row is >= 128 bytes and holds 16 copies of the entry
// (c0 or -c0, c1 2^-10), one per lane of a half-warp at byte 8 (lane & 15), so
// the 16 lanes one LDS.64 wavefront serves always hit 16 different bank pairs.
// The address is one LOP3, (h & mask) | lane_off, and rows 0 .. 2^b - 1 (E5 = 0)
// are never addressed, so `lane_off` carries the table base less those rows.
// Same exactness conditions as the signed table (c1 2^-10 exact, no z == 0).
constexpr int kLaneBlockLog2 = 9;                              // 512 threads per CTA
constexpr int kLaneBlock = 1 << kLaneBlockLog2;
constexpr int kLaneTableBytes = 55 << 10;                      // rows 2^b .. (56 << b) - 1: 56320 for every b
constexpr int kLaneScratch = kLaneTableBytes + 16;             // after the CTA state slot: the parked entries
constexpr int kLaneBytes = kLaneScratch + 8 * (23 << 4);       // dynamic shared memory per CTA (b <= 4)
constexpr int kLaneMaxBits = 4;                                // b = 4: 8 copies (2-way conflicts at worst)

template <bool OR>  // the table's row 0 is at shared address 0: (h & mask) | lane_base is the address
struct EvalLinLane {
    uint32_t lane_base;  // shared byte address of row 0 plus this lane's copy offset
    uint32_t mask;       // 0xFFFF << (10 - b) & 0xFFFF
    __device__ __forceinline__ uint32_t addr(uint32_t h) const {
        // rows E5 = 1 .. 23 of either sign: byte offsets [1 KB, 24 KB) and [33 KB, 56 KB) from row 0
        ARV_DCHECK(((h & mask) & 0x7FFFu) >= 1024u && ((h & mask) & 0x7FFFu) < 24576u);
        return OR ? ((h & mask) | lane_base) : ((h & mask) + lane_base);
    }
    __device__ __forceinline__ static uint32_t magic(uint32_t w) {
        return 0x44C00000u + static_cast<uint32_t>(static_cast<int32_t>(w) >> 9);  // (12582912 + i) 2^-13
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        const float vh = __fadd_rn(__fadd_rn(__uint_as_float(magic(w)), -1536.0f), 0x1p-14f);
        uint32_t h;
        asm("{.reg .b16 t; cvt.rz.f16.f32 t, %1; mov.b32 %0, {t, 0};}" : "=r"(h) : "f"(vh));
        const float2 c = lds_f32x2(addr(h));
        return __float_as_uint(__fadd_rn(__fmul_rn(c.y, vh), c.x));
    }
    static constexpr bool kHasPair = true;
    __device__ __forceinline__ void pair(uint32_t w0, uint32_t w1, uint32_t &r0, uint32_t &r1) const {
        const uint64_t g = pack2(magic(w0), magic(w1));
        const uint64_t vh = f32x2_add(f32x2_add(g, kMinusMagic2), kHalf2);
        const float v0 = __uint_as_float(lo32(vh)), v1 = __uint_as_float(hi32(vh));
        uint32_t h;  // {f16(v1), f16(v0)}, truncated
        asm("cvt.rz.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(v1), "f"(v0));
        const float2 c0 = lds_f32x2(addr(h));
        const float2 c1 = lds_f32x2(addr(h >> 16));
        r0 = __float_as_uint(__fadd_rn(__fmul_rn(c0.y, v0), c0.x));
        r1 = __float_as_uint(__fadd_rn(__fmul_rn(c1.y, v1), c1.x));
    }
    static constexpr uint64_t kMinusMagic2 = 0xC4C00000C4C00000ull;  // {-1536, -1536}
    static constexpr uint64_t kHalf2 = 0x3880000038800000ull;        // {2^-14, 2^-14}
};

// Stage the lane table (`sm` points at row 2^b: the E5 = 0 rows are not
// allocated); verdict as stage_linsigned.  Two phases so that the stores are
// conflict-free: the (23 << b) entries are checked and parked in `scratch`
// (one per thread), then every thread writes copy (i % copies) of entry
// (i / copies) -- consecutive lanes fill consecutive 8-byte slots of a row.
__device__ __forceinline__ bool stage_linlane(char *sm, float2 *scratch, const float *__restrict__ coeffs, int K, int b) {
    const int row_bytes = 1 << (10 - b);
    const int copies = row_bytes >= 128 ? 16 : row_bytes / 8;
    const int n_entries = 23 << b;
    bool ok = true;
    for (int e = threadIdx.x; e < n_entries; e += blockDim.x) {
        float c0, c1s;
        ok &= linsigned_entry(coeffs, K, b, e, 0x1p-10f, c0, c1s);
        scratch[e] = make_float2(c0, c1s);
    }
    ok = __syncthreads_and(ok) != 0;
    for (int i = threadIdx.x; i < n_entries * copies; i += blockDim.x) {
        const int e = i / copies, c = i - e * copies;
        ARV_DCHECK(e < n_entries && (static_cast<size_t>(e) + (32 << b) + 1) * row_bytes <= kLaneTableBytes);
        const float2 v = scratch[e];
        // e = (E5 - 1) << b | sub; row (E5 << b | sub) = e + 2^b, stored less the 2^b skipped rows
        reinterpret_cast<float2 *>(sm + static_cast<size_t>(e) * row_bytes)[c] = v;
        reinterpret_cast<float2 *>(sm + (static_cast<size_t>(e) + (32 << b)) * row_bytes)[c] = make_float2(-v.x, v.y);
    }
    __syncthreads();
    return ok;
}

// --------------------------------------------------------------- kernels --
template <int MODE, class Eval>
__global__ void __launch_bounds__(256, ARV_GEN_MINB) k_gen_simple(GenArgs a, uint32_t *out, Eval eval) {
    gen_dispatch<MODE>(a, out, eval);
}

// KIND: 0 = table in shared memory (q <= 14), 1 = global (q <= 23), 2 = global, q = 24.
template <int MODE, int KIND>
__global__ void __launch_bounds__(256, ARV_GEN_MINB) k_pcg32_constant(GenArgs a, const float *__restrict__ values, int q,
                                                        uint32_t *out) {
#if ARV_GEN_PDL
    // let the next kernel on the stream start its CTAs (start-state walk) as ours retire;
    // our own table reads and stores come after griddepcontrol.wait (gen_loop_vec)
    asm volatile("griddepcontrol.launch_dependents;");
#endif
    if constexpr (KIND == 0) {
        extern __shared__ float4 smem4[];
        float *sm = reinterpret_cast<float *>(smem4);
        const int nv = 1 << q;
        const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
        gen_dispatch<MODE>(a, out, EvalConstantSmem{base, 32 - q, 4u + threadIdx.x * a.zero32}, [&] {
            for (int i = threadIdx.x; i < nv; i += blockDim.x) sm[i] = __ldg(values + i);
            __syncthreads();
        });
    } else if constexpr (KIND == 1) {
        gen_dispatch<MODE>(a, out, EvalConstantGlobal{values, 32 - q});
    } else {
        gen_dispatch<MODE>(a, out, EvalConstant24{values});
    }
}

template <int DEG, int MODE>
__global__ void __launch_bounds__(256, ARV_GEN_MINB) k_pcg32_subdyadic(GenArgs a, const float *__restrict__ coeffs, int K, int b,
                                                         uint32_t *out) {
#if ARV_GEN_PDL
    // let the next kernel on the stream start its CTAs as ours retire
    asm volatile("griddepcontrol.launch_dependents;");
#endif
    __shared__ float sm[(DEG + 1) * kLatticePlane];
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) - 4u * (kLatticeE0 << b);
    // the table is staged after griddepcontrol.wait (see gen_loop_vec)
    gen_dispatch<MODE>(a, out, EvalSubDyadic<DEG>{base, 23 - b, 4u + threadIdx.x * a.zero32},
                       [&] { stage_subdyadic<DEG>(sm, coeffs, K, b); });
}

// Degree-1 sub-interval generator on the signed table (EvalLinSigned), with
// EvalSubDyadic<1> as the exact fallback for tables that fail its checks.
template <int MODE>
__global__ void __launch_bounds__(256, ARV_GEN_MINB) k_pcg32_linsigned(GenArgs a, const float *__restrict__ coeffs, int K,
                                                                      int b, uint32_t *out) {
    static_assert(MODE == 4 || MODE == 8, "vector stores only");
#if ARV_GEN_PDL
    asm volatile("griddepcontrol.launch_dependents;");
#endif
    extern __shared__ float4 smem4[];
    const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t s = group_start<>(a, g0);
    pdl_wait();
    float2 *tab = reinterpret_cast<float2 *>(smem4);
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
    if (stage_linsigned(tab, coeffs, K, b)) {
        // not unrolled: 182.0 vs 184.7 us (unroll 2) / 188.9 us (unroll 4) at 2^28,
        // sustained 210.3 vs 211.3 / 216.4 us (tools/gen_tune.py)
        gen_run<MODE, kSignedUnroll>(a, out, EvalLinSigned{sbase - 8u * (kSignedE0 << b), 23 - b,
                                                           8u + threadIdx.x * a.zero32}, s, g0);
    } else {  // CTA-uniform
        float *sm = reinterpret_cast<float *>(smem4);
        __syncthreads();
        stage_subdyadic<1>(sm, coeffs, K, b);
        gen_run<MODE>(a, out, EvalSubDyadic<1>{sbase - 4u * (kLatticeE0 << b), 23 - b, 4u + threadIdx.x * a.zero32}, s,
                      g0);
    }
}

// The headline kernel for large calls: lane-private table copies, 512 threads
// per CTA (3 CTAs per SM share 168 KB of tables).  Tables failing the
// exactness checks fall back to EvalSubDyadic<1> like k_pcg32_linsigned.
template <int MODE>
__global__ void __launch_bounds__(kLaneBlock, 3) k_pcg32_linlane(GenArgs a, const float *__restrict__ coeffs, int K, int b,
                                                                 uint32_t *out) {
    static_assert(MODE == 4 || MODE == 8, "vector stores only");
#if ARV_GEN_PDL
    asm volatile("griddepcontrol.launch_dependents;");
#endif
    // No static shared memory in this kernel: the table is the first thing in
    // the CTA's window, behind the 1 KB the driver reserves -- exactly the
    // 2^b unaddressed rows (1 KB for every b), so row 0 sits at shared address
    // 0 and the lookup address needs no base add.  Checked at run time; any
    // other placement takes the variant with the add.
    extern __shared__ float4 smem4[];
    char *tab = reinterpret_cast<char *>(smem4);
    const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t s = group_start<kLaneBlockLog2>(a, g0, *reinterpret_cast<uint64_t *>(tab + kLaneTableBytes));
    pdl_wait();
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
    if (stage_linlane(tab, reinterpret_cast<float2 *>(tab + kLaneScratch), coeffs, K, b)) {
        const uint32_t row_bytes = 1u << (10 - b);
        const uint32_t copies = row_bytes >= 128 ? 16 : row_bytes / 8;
        const uint32_t lane_base = sbase - 1024u + 8u * (threadIdx.x & (copies - 1));  // 2^b rows = 1 KB
        uint32_t mask = (0xFFFFu << (10 - b)) & 0xFFFFu;
        asm volatile("mov.b32 %0, %0;" : "+r"(mask));  // opaque: one LOP3 (h & mask) | lane_base per lookup
        if (sbase == 1024u) gen_run<MODE, kSignedUnroll>(a, out, EvalLinLane<true>{lane_base, mask}, s, g0);
        else gen_run<MODE, kSignedUnroll>(a, out, EvalLinLane<false>{lane_base, mask}, s, g0);
    } else {  // CTA-uniform
        float *sm = reinterpret_cast<float *>(smem4);
        __syncthreads();
        stage_subdyadic<1>(sm, coeffs, K, b);
        gen_run<MODE>(a, out, EvalSubDyadic<1>{sbase - 4u * (kLatticeE0 << b), 23 - b, 4u + threadIdx.x * a.zero32}, s,
                      g0);
    }
}

// Test hook: every point of the f32 lattice through the generators'
// evaluators (same structs, same staging), out[k] = eval(w), w >> 9 == k.
// The low 9 bits of w are set to a hash of k: the evaluators must ignore them.
constexpr int kLatticeN = 1 << 23;
template <int MODE>
__global__ void __launch_bounds__(256) k_lattice_sub(const float *__restrict__ coeffs, int K, int b, uint32_t *out,
                                                     int *fast) {
    extern __shared__ float4 smem4[];
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem4));
    const int stride = gridDim.x * blockDim.x;
    const int k0 = blockIdx.x * blockDim.x + threadIdx.x;
    bool use_signed = false;
    if constexpr (MODE == 1) {
        use_signed = stage_linsigned(reinterpret_cast<float2 *>(smem4), coeffs, K, b);
        if (fast && blockIdx.x == 0 && threadIdx.x == 0) *fast = use_signed ? 1 : 0;
    }
    if constexpr (MODE == 2) {
        char *tab = reinterpret_cast<char *>(smem4);
        const bool lane_ok = stage_linlane(tab, reinterpret_cast<float2 *>(tab + kLaneScratch), coeffs, K, b);
        if (fast && blockIdx.x == 0 && threadIdx.x == 0) *fast = lane_ok ? 1 : 0;
        if (lane_ok) {
            const uint32_t row_bytes = 1u << (10 - b);
            const uint32_t copies = row_bytes >= 128 ? 16 : row_bytes / 8;
            const EvalLinLane<false> ev{sbase - 1024u + 8u * (threadIdx.x & (copies - 1)), (0xFFFFu << (10 - b)) & 0xFFFFu};
            // pairs through pair() (the generator's path), the odd point out through operator()
            for (int k = 2 * k0; k < kLatticeN; k += 2 * stride) {
                const uint32_t w0 = (static_cast<uint32_t>(k) << 9) | ((k * 0x9E3779B1u) >> 23);
                const uint32_t w1 = (static_cast<uint32_t>(k + 1) << 9) | (((k + 1) * 0x9E3779B1u) >> 23);
                if ((k >> 1) & 1) {
                    ev.pair(w0, w1, out[k], out[k + 1]);
                } else {
                    out[k] = ev(w0);
                    out[k + 1] = ev(w1);
                }
            }
            return;
        }
    }
    if (use_signed) {
        const EvalLinSigned ev{sbase - 8u * (kSignedE0 << b), 23 - b, 8u};
        for (int k = k0; k < kLatticeN; k += stride) out[k] = ev((static_cast<uint32_t>(k) << 9) | ((k * 0x9E3779B1u) >> 23));
        return;
    }
    __syncthreads();
    stage_subdyadic<1>(reinterpret_cast<float *>(smem4), coeffs, K, b);
    const EvalSubDyadic<1> ev{sbase - 4u * (kLatticeE0 << b), 23 - b, 4u};
    for (int k = k0; k < kLatticeN; k += stride) out[k] = ev((static_cast<uint32_t>(k) << 9) | ((k * 0x9E3779B1u) >> 23));
}

// f64 exact comparator: groups of 4 samples, two 16-byte stores.
__global__ void __launch_bounds__(256) k_pcg32_gauss64(GenArgs a, double *__restrict__ out) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t n_full = static_cast<uint64_t>(a.n) >> 2;
    const Affine j0 = lcg_jump(4ull * g, a.inc);
    uint64_t s = j0.a * a.s_base + j0.c;
    for (; g < n_full; g += T) {
        double u[4], r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            u[i] = static_cast<double>(u32_to_f32(pcg32_output(s)));
            s = i < 3 ? lcg_step(s, kPcgMult, a.inc) : lcg_step(s, a.stride.a, a.stride.c);
        }
        as241_f64_batch<4>(u, r);  // tail log/sqrt compacted across the warp
        double2 *o = reinterpret_cast<double2 *>(out + 4 * g);
        __stcs(o, make_double2(r[0], r[1]));
        __stcs(o + 1, make_double2(r[2], r[3]));
    }
    const int rem = static_cast<int>(a.n & 3);
    if (g == n_full && rem) {
        for (int i = 0; i < rem; ++i) {
            out[4 * g + i] = as241_f64(static_cast<double>(u32_to_f32(pcg32_output(s))));
            s = lcg_step(s, kPcgMult, a.inc);
        }
    }
}

// Write-only roof probes: MODE 4 = st.global.cs.v4, 8 = st.global.cs.v8,
// 5 = st.global.v4 (default eviction).
template <int MODE>
__global__ void __launch_bounds__(256) k_store_probe(uint32_t *out, int64_t n) {
    const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
    constexpr int G = MODE == 8 ? 8 : 4;
    uint32_t r[G];
#pragma unroll
    for (int i = 0; i < G; ++i) r[i] = 0x3F800000u + i;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n / G; i += T) {
        if constexpr (MODE == 5)
            *reinterpret_cast<uint4 *>(out + G * i) = make_uint4(r[0], r[1], r[2], r[3]);
        else
            VecOut<G>::store(out + G * i, r);
    }
}

// ------------------------------------------------------------- launchers --
constexpr int kGenBlock = 256;

static bool aligned(const void *p, int bytes) { return (reinterpret_cast<uintptr_t>(p) & (bytes - 1)) == 0; }

// Store mode for an output pointer: the tuned group size if aligned for it.
static int store_mode(const void *out) {
    if (g_group == 8 && aligned(out, 32)) return 8;
    if (aligned(out, 16)) return 4;
    return 1;
}

// One wave: CTAs per SM = the kernel's resident count (a second partial wave
// of a grid-stride kernel cost 2-7% at 2^28 in an earlier build, tools/sweep_launch.py), fewer
// for small n so that every thread keeps >= kMinPerThread samples to amortise
// its jump-ahead (2^24: 4 CTAs/SM beat 8 by 7%; 2^20: 1-2 beat 8 by 30%).
constexpr int64_t kMinPerThread = 64;

// Very large calls (>= 16 one-wave grids of 64 samples per thread, e.g. 2^28
// samples) run 5/3 waves instead: the generators then finish 1.2-1.7% sooner
// (2^28: sub-interval 0.1935 -> 0.1911 ms, constant 0.1663 -> 0.1635 ms;
// 2^26 and below keep one wave, where the extra CTAs cost 2-20%).
static int gen_grid(const void *fn, int64_t n, int mode, size_t smem = 0, int block = kGenBlock,
                    bool extra_wave = true) {
    int per_sm = g_ctas_per_sm;
    if (per_sm <= 0) {
        const int64_t want = n / (static_cast<int64_t>(device_sm_count()) * block * kMinPerThread);
        const int occ = resident_ctas(fn, block, smem);
        per_sm = static_cast<int>(want < 1 ? 1 : (want < occ ? want : occ));
        if (extra_wave && want >= 16 * occ) per_sm = occ + (2 * occ) / 3;
    }
    return stream_grid((n + mode - 1) / mode, block, per_sm);
}

template <class Eval>
static int launch_simple(uint64_t seed, uint64_t sid, uint64_t offset, uint32_t *out, int64_t n, void *stream,
                         Eval ev, const char *what) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "%s: negative n", what);
    if (n == 0) return ARV_OK;
    const int mode = store_mode(out);
    const void *fn = mode == 8   ? (const void *)k_gen_simple<8, Eval>
                     : mode == 4 ? (const void *)k_gen_simple<4, Eval>
                                 : (const void *)k_gen_simple<1, Eval>;
    const int grid = gen_grid(fn, n, mode);
    const int64_t T = static_cast<int64_t>(grid) * kGenBlock;
    const GenArgs a = make_gen_args(seed, sid, offset, n, T, mode == 1 ? 4 : mode);
    cudaStream_t s = as_stream(stream);
    if (mode == 8) k_gen_simple<8, Eval><<<grid, kGenBlock, 0, s>>>(a, out, ev);
    else if (mode == 4) k_gen_simple<4, Eval><<<grid, kGenBlock, 0, s>>>(a, out, ev);
    else k_gen_simple<1, Eval><<<grid, kGenBlock, 0, s>>>(a, out, ev);
    note_launch();
    return check_launch(what);
}

// Degree 1 with b <= kSignedMaxBits runs the signed-table kernel (b = 5
// would need 71 KB of shared memory per CTA).
#ifndef ARV_GEN_SIGNED
#define ARV_GEN_SIGNED 1
#endif
constexpr int kSignedMaxBits = 4;

template <int D>
static void launch_subdyadic(uint64_t seed, uint64_t sid, uint64_t offset, const float *coeffs, int K, int sub_bits,
                             float *out, int64_t n, int mode, void *stream) {
    const bool signed_tab = ARV_GEN_SIGNED && D == 1 && mode != 1 && sub_bits <= kSignedMaxBits;
    // Large calls: the lane-private table (57 KB staged per 512-thread CTA pays
    // off from 2^26 samples on; g_lane_min_n, ARV_TUNE_LANE_MIN_N).
    if (signed_tab && sub_bits <= kLaneMaxBits && g_lane_min_n >= 0 && n >= g_lane_min_n) {
        const void *lfn = mode == 8 ? (const void *)k_pcg32_linlane<8> : (const void *)k_pcg32_linlane<4>;
        // per call: the attribute is per device, and a call of >= 2^26 samples does not notice it
        cudaFuncSetAttribute(lfn, cudaFuncAttributeMaxDynamicSharedMemorySize, kLaneBytes);
        // one wave of 3 CTAs per SM: 174.3 us vs 175.5 us for 5/3 waves at 2^28 (tools/gen_tune_lane.py)
        const int grid = gen_grid(lfn, n, mode, kLaneBytes, kLaneBlock, false);
        const GenArgs a = make_gen_args(seed, sid, offset, n, static_cast<int64_t>(grid) * kLaneBlock, mode);
        uint32_t *o = reinterpret_cast<uint32_t *>(out);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kLaneBlock);
        cfg.dynamicSmemBytes = kLaneBytes;
        cfg.stream = as_stream(stream);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = ARV_GEN_PDL;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (mode == 8) cudaLaunchKernelEx(&cfg, k_pcg32_linlane<8>, a, coeffs, K, sub_bits, o);
        else cudaLaunchKernelEx(&cfg, k_pcg32_linlane<4>, a, coeffs, K, sub_bits, o);
        return;
    }
    const void *fn = signed_tab  ? (mode == 8 ? (const void *)k_pcg32_linsigned<8> : (const void *)k_pcg32_linsigned<4>)
                     : mode == 8 ? (const void *)k_pcg32_subdyadic<D, 8>
                     : mode == 4 ? (const void *)k_pcg32_subdyadic<D, 4>
                                 : (const void *)k_pcg32_subdyadic<D, 1>;
    const size_t smem = signed_tab ? std::max<size_t>(sizeof(float2) * linsigned_entries(sub_bits),
                                                      sizeof(float) * 2 * kLatticePlane)
                                   : 0;
    const int grid = gen_grid(fn, n, mode, smem);
    const int64_t T = static_cast<int64_t>(grid) * kGenBlock;
    const GenArgs a = make_gen_args(seed, sid, offset, n, T, mode == 1 ? 4 : mode);
    uint32_t *o = reinterpret_cast<uint32_t *>(out);
    cudaStream_t s = as_stream(stream);
#if ARV_GEN_PDL
    if (mode != 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kGenBlock);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (signed_tab && mode == 8) cudaLaunchKernelEx(&cfg, k_pcg32_linsigned<8>, a, coeffs, K, sub_bits, o);
        else if (signed_tab) cudaLaunchKernelEx(&cfg, k_pcg32_linsigned<4>, a, coeffs, K, sub_bits, o);
        else if (mode == 8) cudaLaunchKernelEx(&cfg, k_pcg32_subdyadic<D, 8>, a, coeffs, K, sub_bits, o);
        else cudaLaunchKernelEx(&cfg, k_pcg32_subdyadic<D, 4>, a, coeffs, K, sub_bits, o);
        return;
    }
#endif
    if (signed_tab) {
        if (mode == 8) k_pcg32_linsigned<8><<<grid, kGenBlock, smem, s>>>(a, coeffs, K, sub_bits, o);
        else k_pcg32_linsigned<4><<<grid, kGenBlock, smem, s>>>(a, coeffs, K, sub_bits, o);
        return;
    }
    if (mode == 8) k_pcg32_subdyadic<D, 8><<<grid, kGenBlock, 0, s>>>(a, coeffs, K, sub_bits, o);
    else if (mode == 4) k_pcg32_subdyadic<D, 4><<<grid, kGenBlock, 0, s>>>(a, coeffs, K, sub_bits, o);
    else k_pcg32_subdyadic<D, 1><<<grid, kGenBlock, 0, s>>>(a, coeffs, K, sub_bits, o);
}

}  // namespace arv

using namespace arv;

extern "C" {

int arv_set_tuning(int key, int value) {
    switch (key) {
        case ARV_TUNE_GROUP:
            if (value != 4 && value != 8) return set_error(ARV_ERR_CONFIG, "group must be 4 or 8");
            g_group = value;
            return ARV_OK;
        case ARV_TUNE_CIR_SEGMENT:
            if (value < 0) return set_error(ARV_ERR_CONFIG, "cir segment must be >= 0");
            g_cir_segment = value;
            return ARV_OK;
        case ARV_TUNE_GBM_KERNEL:
            if (value != 0 && value != 2 && value != 3) return set_error(ARV_ERR_CONFIG, "gbm kernel must be 0, 2 or 3");
            g_gbm_kernel = value;
            return ARV_OK;
        case ARV_TUNE_LANE_MIN_N:  // log2 of the smallest call that takes the lane-table kernel; < 0: never
            if (value > 40) return set_error(ARV_ERR_CONFIG, "lane_min_n (log2) must be <= 40");
            g_lane_min_n = value < 0 ? -1 : (int64_t{1} << value);
            return ARV_OK;
        case ARV_TUNE_NC_CERTIFY:
            return set_nc_certify(value);
        case ARV_TUNE_CTAS_PER_SM:
            if (value < 0 || value > 32) return set_error(ARV_ERR_CONFIG, "ctas_per_sm must be in [0 (auto), 32]");
            g_ctas_per_sm = value;
            return ARV_OK;
        default:
            return set_error(ARV_ERR_CONFIG, "unknown tuning key %d", key);
    }
}

int arv_pcg32_words(uint64_t seed, uint64_t stream_id, uint64_t offset, uint32_t *out, int64_t n, void *stream) {
    return launch_simple(seed, stream_id, offset, out, n, stream, EvalWord{}, "arv_pcg32_words");
}

int arv_pcg32_uniform_f32(uint64_t seed, uint64_t stream_id, uint64_t offset, float *out, int64_t n,
                          void *stream) {
    return launch_simple(seed, stream_id, offset, reinterpret_cast<uint32_t *>(out), n, stream, EvalUniform{},
                         "arv_pcg32_uniform_f32");
}

int arv_pcg32_gaussian_f32(uint64_t seed, uint64_t stream_id, uint64_t offset, float *out, int64_t n,
                           void *stream) {
    return launch_simple(seed, stream_id, offset, reinterpret_cast<uint32_t *>(out), n, stream, EvalGauss32{},
                         "arv_pcg32_gaussian_f32");
}

int arv_pcg32_constant_f32(uint64_t seed, uint64_t stream_id, uint64_t offset, const float *values, int q,
                           float *out, int64_t n, void *stream) {
    if (q < 1 || q > 24) return set_error(ARV_ERR_CONFIG, "interval exponent q must be in [1, 24], got %d", q);
    if (n < 0) return set_error(ARV_ERR_CONFIG, "negative n");
    if (n == 0) return ARV_OK;
    const int kind = q <= 14 ? 0 : (q <= 23 ? 1 : 2);
    const size_t smem = kind == 0 ? (sizeof(float) << q) : 0;
    const int mode = store_mode(out);
#define ARV_CONST_FN(M) \
    (kind == 0 ? (const void *)k_pcg32_constant<M, 0> : kind == 1 ? (const void *)k_pcg32_constant<M, 1> : (const void *)k_pcg32_constant<M, 2>)
    const void *fn = mode == 8 ? ARV_CONST_FN(8) : mode == 4 ? ARV_CONST_FN(4) : ARV_CONST_FN(1);
#undef ARV_CONST_FN
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = gen_grid(fn, n, mode, smem);
    const int64_t T = static_cast<int64_t>(grid) * kGenBlock;
    const GenArgs a = make_gen_args(seed, stream_id, offset, n, T, mode == 1 ? 4 : mode);
    uint32_t *o = reinterpret_cast<uint32_t *>(out);
    void *args[] = {(void *)&a, (void *)&values, (void *)&q, (void *)&o};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGenBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (ARV_GEN_PDL && mode != 1) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
    note_launch();
    return check_launch("arv_pcg32_constant_f32");
}

int arv_pcg32_subdyadic_f32(uint64_t seed, uint64_t stream_id, uint64_t offset, const float *coeffs, int degree,
                            int K, int sub_bits, float *out, int64_t n, void *stream) {
    if (degree < 1 || degree > 5) return set_error(ARV_ERR_CONFIG, "polynomial degree must be in [1, 5], got %d", degree);
    if (K < 1 || K > 40) return set_error(ARV_ERR_CONFIG, "octave count K must be in [1, 40], got %d", K);
    if (sub_bits < 0 || sub_bits > 5) return set_error(ARV_ERR_CONFIG, "sub_bits must be in [0, 5], got %d", sub_bits);
    if (n < 0) return set_error(ARV_ERR_CONFIG, "negative n");
    if (n == 0) return ARV_OK;
    const int mode = store_mode(out);
    switch (degree) {
        case 1: launch_subdyadic<1>(seed, stream_id, offset, coeffs, K, sub_bits, out, n, mode, stream); break;
        case 2: launch_subdyadic<2>(seed, stream_id, offset, coeffs, K, sub_bits, out, n, mode, stream); break;
        case 3: launch_subdyadic<3>(seed, stream_id, offset, coeffs, K, sub_bits, out, n, mode, stream); break;
        case 4: launch_subdyadic<4>(seed, stream_id, offset, coeffs, K, sub_bits, out, n, mode, stream); break;
        default: launch_subdyadic<5>(seed, stream_id, offset, coeffs, K, sub_bits, out, n, mode, stream); break;
    }
    note_launch();
    return check_launch("arv_pcg32_subdyadic_f32");
}

int arv_lattice_subdyadic_f32(const float *coeffs, int degree, int K, int sub_bits, int mode, float *out, int *fast,
                              void *stream) {
    if (degree != 1) return set_error(ARV_ERR_CONFIG, "lattice hook: degree must be 1");
    if (K < 1 || K > 40) return set_error(ARV_ERR_CONFIG, "octave count K must be in [1, 40], got %d", K);
    if (sub_bits < 0 || sub_bits > (mode == 1 ? kSignedMaxBits : mode == 2 ? kLaneMaxBits : 5))
        return set_error(ARV_ERR_CONFIG, "sub_bits out of range for mode %d", mode);
    const size_t smem = std::max<size_t>({sizeof(float2) * linsigned_entries(sub_bits), sizeof(float) * 2 * kLatticePlane,
                                          mode == 2 ? size_t{kLaneBytes} : size_t{0}});
    cudaStream_t s = as_stream(stream);
    uint32_t *o = reinterpret_cast<uint32_t *>(out);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute((const void *)k_lattice_sub<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute((const void *)k_lattice_sub<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute((const void *)k_lattice_sub<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (mode == 2) k_lattice_sub<2><<<2 * device_sm_count(), 256, smem, s>>>(coeffs, K, sub_bits, o, fast);
    else if (mode == 1) k_lattice_sub<1><<<4 * device_sm_count(), 256, smem, s>>>(coeffs, K, sub_bits, o, fast);
    else k_lattice_sub<0><<<4 * device_sm_count(), 256, smem, s>>>(coeffs, K, sub_bits, o, fast);
    note_launch();
    return check_launch("arv_lattice_subdyadic_f32");
}

int arv_pcg32_gaussian_f64(uint64_t seed, uint64_t stream_id, uint64_t offset, double *out, int64_t n, void *stream) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "negative n");
    if (n == 0) return ARV_OK;
    if (!aligned(out, 16)) return set_error(ARV_ERR_CONFIG, "arv_pcg32_gaussian_f64: out must be 16-byte aligned");
    const int grid = gen_grid((const void *)k_pcg32_gauss64, n, 4);
    const int64_t T = static_cast<int64_t>(grid) * kGenBlock;
    const GenArgs a = make_gen_args(seed, stream_id, offset, n, T, 4);
    k_pcg32_gauss64<<<grid, kGenBlock, 0, as_stream(stream)>>>(a, out);
    note_launch();
    return check_launch("arv_pcg32_gaussian_f64");
}

int arv_store_probe_ex(float *out, int64_t n, int mode, void *stream) {
    if (n < 0 || (n & 7) || !aligned(out, 32)) return set_error(ARV_ERR_CONFIG, "store probe needs n % 8 == 0 and 32B alignment");
    if (n == 0) return ARV_OK;
    const int G = mode == 8 ? 8 : 4;
    const int grid = gen_grid((const void *)k_store_probe<8>, n, G);
    uint32_t *o = reinterpret_cast<uint32_t *>(out);
    cudaStream_t s = as_stream(stream);
    if (mode == 8) k_store_probe<8><<<grid, kGenBlock, 0, s>>>(o, n);
    else if (mode == 5) k_store_probe<5><<<grid, kGenBlock, 0, s>>>(o, n);
    else k_store_probe<4><<<grid, kGenBlock, 0, s>>>(o, n);
    note_launch();
    return check_launch("arv_store_probe_ex");
}

int arv_store_probe(float *out, int64_t n, void *stream) { return arv_store_probe_ex(out, n, 8, stream); }

}  // extern "C"

// Fused PCG32 -> inverse-CDF generators.
//
// One thread owns a PCG32 state in registers and produces groups of four
// consecutive samples 4g..4g+3 (g = its group index), so each warp store is a
// fully coalesced 512-byte st.global.v4; the only HBM traffic is the output.
// Within a group the LCG steps once per sample; between groups the thread
// jumps over the 4(T-1) samples the other T-1 threads own with one affine
// map (A, C) = LCG^(4T-3), precomputed on the host.  Output i of the call is
// PCG32 output (offset + i) of stream (seed, stream_id) whatever the grid,
// so shards on different GPUs concatenate bit-exactly.
//
// Evaluators (reference semantics, see oracle/oracle.c):
//   constant   values[floor(2^q u)]            (_kernels.pyx:16-23)
//   subdyadic  octave x sub-interval Horner    (_kernels.pyx:76-93 when sub_bits = 0)
//   uniform    u itself; gaussian32/64 = AS241 (exact_dist.py:87-126)
#include "arv_common.cuh"

namespace arv {

struct GenArgs {
    uint64_t s_base;  // state whose output is sample 0 of this call
    uint64_t inc;
    Affine stride;    // LCG^(4T-3)
    int64_t n;
};

static GenArgs make_gen_args(uint64_t seed, uint64_t stream_id, uint64_t offset, int64_t n,
                             int64_t total_threads) {
    const StreamStart st = pcg32_start(seed, stream_id, offset);
    GenArgs a;
    a.s_base = st.state;
    a.inc = st.inc;
    a.stride = lcg_jump(4ull * static_cast<uint64_t>(total_threads) - 3ull, st.inc);
    a.n = n;
    return a;
}

// Drive `eval(w) -> uint32 bits` over the call's samples with v4 stores.
template <class Eval>
__device__ __forceinline__ void gen_loop_v4(const GenArgs &a, uint32_t *__restrict__ out, const Eval &eval) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t n_full = static_cast<uint64_t>(a.n) >> 2;
    const Affine j0 = lcg_jump(4ull * g, a.inc);
    uint64_t s = j0.a * a.s_base + j0.c;
    const uint64_t inc = a.inc;
    const Affine st = a.stride;
    for (; g < n_full; g += T) {
        const uint32_t w0 = pcg32_output(s);
        s = s * kPcgMult + inc;
        const uint32_t w1 = pcg32_output(s);
        s = s * kPcgMult + inc;
        const uint32_t w2 = pcg32_output(s);
        s = s * kPcgMult + inc;
        const uint32_t w3 = pcg32_output(s);
        s = st.a * s + st.c;
        uint4 r;
        r.x = eval(w0);
        r.y = eval(w1);
        r.z = eval(w2);
        r.w = eval(w3);
        __stcs(reinterpret_cast<uint4 *>(out) + g, r);
    }
    const int rem = static_cast<int>(a.n & 3);
    if (g == n_full && rem) {
        for (int i = 0; i < rem; ++i) {
            out[4 * g + i] = eval(pcg32_output(s));
            s = s * kPcgMult + inc;
        }
    }
}

// Scalar-store variant for outputs that are not 16-byte aligned.
template <class Eval>
__device__ __forceinline__ void gen_loop_v1(uint64_t s_base, uint64_t inc, Affine strideT, int64_t n,
                                            uint32_t *__restrict__ out, const Eval &eval) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const Affine j0 = lcg_jump(i, inc);
    uint64_t s = j0.a * s_base + j0.c;
    for (; i < static_cast<uint64_t>(n); i += T) {
        out[i] = eval(pcg32_output(s));
        s = strideT.a * s + strideT.c;
    }
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
// 2k + 1 for q = 24.  Table in shared memory (q <= 14) or global (L2).
struct EvalConstant {
    const float *tab;
    int shift;  // 32 - q, or -1 for q == 24
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        const uint32_t idx = shift >= 0 ? (w >> shift) : (((w >> 9) << 1) | 1u);
        return __float_as_uint(tab[idx]);
    }
};
// Octave x sub-interval, reversed table (row r = K - j, r = K is the zero
// row of v = 1/2): entry = (bits(v) >> (23 - b)) - ((126 - K) << b),
// clamped below at 0 (all octaves >= K share the singular row 0).
template <int DEG>
struct EvalSubDyadic {
    const float *tab;  // (DEG+1) planes of `plane` floats, or float2 pairs when DEG == 1
    int shift, base, plane;
    __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
        const Reflected r = reflect_u32(w);
        const int e = max(static_cast<int>(__float_as_uint(r.v) >> shift) - base, 0);
        float z;
        if constexpr (DEG == 1) {
            const float2 c = reinterpret_cast<const float2 *>(tab)[e];
            z = __fadd_rn(__fmul_rn(c.y, r.v), c.x);
        } else {
            z = tab[DEG * plane + e];
#pragma unroll
            for (int d = DEG - 1; d >= 0; --d) z = __fadd_rn(__fmul_rn(z, r.v), tab[d * plane + e]);
        }
        return __float_as_uint(z) ^ (r.m & 0x80000000u);
    }
};

// Stage the natural-layout table (DEG+1, K, nsub) into the reversed layout.
template <int DEG>
__device__ __forceinline__ void stage_subdyadic(float *sm, const float *__restrict__ coeffs, int K, int b) {
    const int nsub = 1 << b;
    const int plane = (K + 1) << b;
    for (int e = threadIdx.x; e < plane; e += blockDim.x) {
        const int r = e >> b, s = e & (nsub - 1);
        const int j = K - r;
        for (int d = 0; d <= DEG; ++d) {
            const float c = j == 0 ? 0.0f : __ldg(coeffs + (static_cast<int64_t>(d) * K + (j - 1)) * nsub + (j == K ? 0 : s));
            if constexpr (DEG == 1) sm[2 * e + d] = c;
            else sm[d * plane + e] = c;
        }
    }
    __syncthreads();
}

// --------------------------------------------------------------- kernels --
template <class Eval>
__global__ void __launch_bounds__(256) k_gen_simple(GenArgs a, uint32_t *out, Eval eval) {
    gen_loop_v4(a, out, eval);
}
template <class Eval>
__global__ void __launch_bounds__(256) k_gen_simple_v1(uint64_t s_base, uint64_t inc, Affine strideT, int64_t n,
                                                       uint32_t *out, Eval eval) {
    gen_loop_v1(s_base, inc, strideT, n, out, eval);
}

template <bool V4>
__global__ void __launch_bounds__(256) k_pcg32_constant(GenArgs a, const float *__restrict__ values, int q,
                                                        int use_smem, uint32_t *out) {
    extern __shared__ float4 smem4[];
    float *sm = reinterpret_cast<float *>(smem4);
    const float *tab = values;
    if (use_smem) {
        const int nv = 1 << q;
        for (int i = threadIdx.x; i < nv; i += blockDim.x) sm[i] = __ldg(values + i);
        __syncthreads();
        tab = sm;
    }
    EvalConstant ev{tab, q <= 23 ? 32 - q : -1};
    if constexpr (V4) {
        gen_loop_v4(a, out, ev);
    } else {
        const Affine sT = lcg_jump(static_cast<uint64_t>(gridDim.x) * blockDim.x, a.inc);
        gen_loop_v1(a.s_base, a.inc, sT, a.n, out, ev);
    }
}

template <int DEG, bool V4>
__global__ void __launch_bounds__(256) k_pcg32_subdyadic(GenArgs a, const float *__restrict__ coeffs, int K, int b,
                                                         uint32_t *out) {
    extern __shared__ float4 smem4[];
    float *sm = reinterpret_cast<float *>(smem4);
    stage_subdyadic<DEG>(sm, coeffs, K, b);
    EvalSubDyadic<DEG> ev{sm, 23 - b, (126 - K) << b, (K + 1) << b};
    if constexpr (V4) {
        gen_loop_v4(a, out, ev);
    } else {
        const Affine sT = lcg_jump(static_cast<uint64_t>(gridDim.x) * blockDim.x, a.inc);
        gen_loop_v1(a.s_base, a.inc, sT, a.n, out, ev);
    }
}

// f64 exact comparator: groups of 4 samples, two 16-byte stores.
__global__ void __launch_bounds__(256) k_pcg32_gauss64(GenArgs a, double *__restrict__ out) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t n_full = static_cast<uint64_t>(a.n) >> 2;
    const Affine j0 = lcg_jump(4ull * g, a.inc);
    uint64_t s = j0.a * a.s_base + j0.c;
    for (; g < n_full; g += T) {
        double r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            r[i] = as241_f64(static_cast<double>(u32_to_f32(pcg32_output(s))));
            s = i < 3 ? s * kPcgMult + a.inc : a.stride.a * s + a.stride.c;
        }
        double2 *o = reinterpret_cast<double2 *>(out + 4 * g);
        __stcs(o, make_double2(r[0], r[1]));
        __stcs(o + 1, make_double2(r[2], r[3]));
    }
    const int rem = static_cast<int>(a.n & 3);
    if (g == n_full && rem) {
        for (int i = 0; i < rem; ++i) {
            out[4 * g + i] = as241_f64(static_cast<double>(u32_to_f32(pcg32_output(s))));
            s = s * kPcgMult + a.inc;
        }
    }
}

__global__ void __launch_bounds__(256) k_store_probe(float4 *out, int64_t n4) {
    const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += T) __stcs(out + i, v);
}

// ------------------------------------------------------------- launchers --
constexpr int kGenBlock = 256;
constexpr int kGenPerSM = 8;  // 2048 resident threads per SM

static int gen_grid(int64_t n) { return stream_grid((n + 3) / 4, kGenBlock, kGenPerSM); }

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <class Eval>
static int launch_simple(uint64_t seed, uint64_t sid, uint64_t offset, uint32_t *out, int64_t n, void *stream,
                         Eval ev, const char *what) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "%s: negative n", what);
    if (n == 0) return ARV_OK;
    const int grid = gen_grid(n);
    const int64_t T = static_cast<int64_t>(grid) * kGenBlock;
    const GenArgs a = make_gen_args(seed, sid, offset, n, T);
    if (aligned16(out)) {
        k_gen_simple<Eval><<<grid, kGenBlock, 0, as_stream(stream)>>>(a, out, ev);
    } else {
        const Affine sT = lcg_jump(static_cast<uint64_t>(T), a.inc);
        k_gen_simple_v1<Eval><<<grid, kGenBlock, 0, as_stream(stream)>>>(a.s_base, a.inc, sT, n, out, ev);
    }
    note_launch();
    return check_launch(what);
}

}  // namespace arv

using namespace arv;

extern "C" {

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
    const int use_smem = q <= 14;
    const size_t smem = use_smem ? (sizeof(float) << q) : 0;
    const int grid = gen_grid(n);
    const int64_t T = static_cast<int64_t>(grid) * kGenBlock;
    const GenArgs a = make_gen_args(seed, stream_id, offset, n, T);
    uint32_t *o = reinterpret_cast<uint32_t *>(out);
    if (aligned16(out)) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_pcg32_constant<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_pcg32_constant<true><<<grid, kGenBlock, smem, as_stream(stream)>>>(a, values, q, use_smem, o);
    } else {
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_pcg32_constant<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_pcg32_constant<false><<<grid, kGenBlock, smem, as_stream(stream)>>>(a, values, q, use_smem, o);
    }
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
    const size_t smem = sizeof(float) * (degree + 1) * ((size_t)(K + 1) << sub_bits);
    const int grid = gen_grid(n);
    const int64_t T = static_cast<int64_t>(grid) * kGenBlock;
    const GenArgs a = make_gen_args(seed, stream_id, offset, n, T);
    uint32_t *o = reinterpret_cast<uint32_t *>(out);
    cudaStream_t s = as_stream(stream);
    const bool v4 = aligned16(out);
#define ARV_SUB_CASE(D)                                                                         \
    case D:                                                                                     \
        if (v4) k_pcg32_subdyadic<D, true><<<grid, kGenBlock, smem, s>>>(a, coeffs, K, sub_bits, o); \
        else k_pcg32_subdyadic<D, false><<<grid, kGenBlock, smem, s>>>(a, coeffs, K, sub_bits, o);   \
        break;
    switch (degree) {
        ARV_SUB_CASE(1)
        ARV_SUB_CASE(2)
        ARV_SUB_CASE(3)
        ARV_SUB_CASE(4)
        ARV_SUB_CASE(5)
    }
#undef ARV_SUB_CASE
    note_launch();
    return check_launch("arv_pcg32_subdyadic_f32");
}

int arv_pcg32_gaussian_f64(uint64_t seed, uint64_t stream_id, uint64_t offset, double *out, int64_t n, void *stream) {
    if (n < 0) return set_error(ARV_ERR_CONFIG, "negative n");
    if (n == 0) return ARV_OK;
    if (!aligned16(out)) return set_error(ARV_ERR_CONFIG, "arv_pcg32_gaussian_f64: out must be 16-byte aligned");
    const int grid = gen_grid(n);
    const int64_t T = static_cast<int64_t>(grid) * kGenBlock;
    const GenArgs a = make_gen_args(seed, stream_id, offset, n, T);
    k_pcg32_gauss64<<<grid, kGenBlock, 0, as_stream(stream)>>>(a, out);
    note_launch();
    return check_launch("arv_pcg32_gaussian_f64");
}

int arv_store_probe(float *out, int64_t n, void *stream) {
    if (n < 0 || (n & 3) || !aligned16(out)) return set_error(ARV_ERR_CONFIG, "store probe needs n % 4 == 0 and 16B alignment");
    if (n == 0) return ARV_OK;
    const int grid = stream_grid(n / 4, kGenBlock, kGenPerSM);
    k_store_probe<<<grid, kGenBlock, 0, as_stream(stream)>>>(reinterpret_cast<float4 *>(out), n / 4);
    note_launch();
    return check_launch("arv_store_probe");
}

}  // extern "C"

"""ctypes/numpy front-end of the C oracle (TEST INFRASTRUCTURE ONLY).

Each wrapper names the reference function it restates; the arithmetic lives
in ``oracle.c`` (see its header for the rounding rules).
"""

from __future__ import annotations

import ctypes as C
import glob
import importlib.util
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

PCG_MULT = 6364136223846793005
MASK64 = (1 << 64) - 1


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    if ref is None:
        ref = os.path.isdir("/root/reference/pkg")
    if ref:
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)


def _load():
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
        os.path.join(_HERE, "oracle.c")
    ):
        build(ref=False)
    return C.CDLL(_LIB_PATH)


lib = _load()

_u64, _i64, _int, _dbl = C.c_uint64, C.c_int64, C.c_int, C.c_double
_p = C.c_void_p


def _sig(name, *args):
    fn = getattr(lib, name)
    fn.argtypes = list(args)
    fn.restype = None
    return fn


_sig("orc_pcg32_seed", _u64, _u64, C.POINTER(_u64), C.POINTER(_u64))
_sig("orc_lcg_jump", _u64, _u64, C.POINTER(_u64), C.POINTER(_u64))
_sig("orc_pcg32_words", _u64, _u64, _u64, _i64, _p)
_sig("orc_u32_to_f32", _p, _i64, _p)
_sig("orc_u32_to_f64", _p, _i64, _p)
_sig("orc_constant_eval", _p, _i64, _p, _p, _i64)
_sig("orc_dyadic_index", _p, _i64, _p, _i64)
_sig("orc_dyadic_index32", _p, _i64, _p, _i64)
_sig("orc_dyadic_eval", _p, _int, _i64, _p, _p, _i64)
_sig("orc_dyadic_eval32", _p, _int, _i64, _p, _p, _i64)
_sig("orc_ncchi2_eval", _p, _i64, _int, _i64, _dbl, _p, _p, _i64, _p, _i64)
_sig("orc_subdyadic_eval32", _p, _int, _int, _int, _p, _p, _i64)
_sig("orc_as241_f64", _p, _p, _i64)
_sig("orc_as241_f32", _p, _p, _i64)
_sig("orc_pcg32_constant_f32", _u64, _u64, _u64, _p, _int, _p, _i64)
_sig("orc_pcg32_subdyadic_f32", _u64, _u64, _u64, _p, _int, _int, _int, _p, _i64)
_sig("orc_pcg32_dyadic_f32", _u64, _u64, _u64, _p, _int, _i64, _p, _i64)
_sig("orc_pcg32_as241_f64", _u64, _u64, _u64, _p, _i64)
_sig("orc_pcg32_as241_f32", _u64, _u64, _u64, _p, _i64)
_sig("orc_gbm_paths", _dbl, _dbl, _dbl, _dbl, _int, _int, _int, _int, _dbl, _p, _int, _i64,
     _u64, _u64, _i64, _i64, _i64, _p, _p, _p, _p)
_sig("orc_cir_euler_paths", _dbl, _dbl, _dbl, _dbl, _dbl, _int, _int, _int, _dbl, _p, _int, _i64,
     _u64, _u64, _i64, _i64, _i64, _p, _p, _p, _p)
_sig("orc_cir_paths", _dbl, _dbl, _dbl, _dbl, _dbl, _int, _int, _int, _int, _dbl, _p, _int, _i64,
     _u64, _u64, _i64, _i64, _i64, _p, _p, _p, _p)


_sig("orc_philox_words", _u64, _u64, _u64, _i64, _p)
_sig("orc_philox_uniforms", _u64, _u64, _u64, _i64, _p)


def philox_words(seed: int, sid: int, counter: int, n: int) -> np.ndarray:
    """UniformStream(seed, sid, counter).raw_words(n) (sampler.py:48-57)."""
    out = np.empty(n, dtype=np.uint64)
    lib.orc_philox_words(seed, sid, counter, n, out.ctypes.data_as(C.c_void_p))
    return out


def philox_uniforms(seed: int, sid: int, counter: int, n: int) -> np.ndarray:
    """UniformStream(seed, sid, counter).uniforms(n) (sampler.py:59-62)."""
    out = np.empty(n, dtype=np.float64)
    lib.orc_philox_uniforms(seed, sid, counter, n, out.ctypes.data_as(C.c_void_p))
    return out


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


# --------------------------------------------------------------------------
# PCG32
# --------------------------------------------------------------------------

def pcg32_seed(initstate: int, initseq: int) -> tuple[int, int]:
    s, inc = _u64(), _u64()
    lib.orc_pcg32_seed(initstate, initseq, C.byref(s), C.byref(inc))
    return s.value, inc.value


def lcg_jump(delta: int, inc: int) -> tuple[int, int]:
    a, c = _u64(), _u64()
    lib.orc_lcg_jump(delta, inc, C.byref(a), C.byref(c))
    return a.value, c.value


def pcg32_words(initstate: int, initseq: int, offset: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    lib.orc_pcg32_words(initstate, initseq, offset, n, _ptr(out))
    return out


def pcg32_words_py(initstate: int, initseq: int, n: int) -> np.ndarray:
    """Independent pure-Python PCG32 (second restatement, small n only)."""
    inc = ((initseq << 1) | 1) & MASK64
    s = 0
    s = (s * PCG_MULT + inc) & MASK64
    s = (s + initstate) & MASK64
    s = (s * PCG_MULT + inc) & MASK64
    out = []
    for _ in range(n):
        old = s
        s = (old * PCG_MULT + inc) & MASK64
        xs = (((old >> 18) ^ old) >> 27) & 0xFFFFFFFF
        rot = old >> 59
        out.append(((xs >> rot) | (xs << ((-rot) & 31))) & 0xFFFFFFFF)
    return np.array(out, dtype=np.uint32)


def u32_to_f32(w) -> np.ndarray:
    w = _c(w, np.uint32)
    out = np.empty(w.shape, dtype=np.float32)
    lib.orc_u32_to_f32(_ptr(w), w.size, _ptr(out))
    return out


def u32_to_f64(w) -> np.ndarray:
    w = _c(w, np.uint32)
    out = np.empty(w.shape, dtype=np.float64)
    lib.orc_u32_to_f64(_ptr(w), w.size, _ptr(out))
    return out


# --------------------------------------------------------------------------
# The six plugin kernels (_kernels.pyx:16-143)
# --------------------------------------------------------------------------

def constant_eval(values, u) -> np.ndarray:
    values = _c(values, np.float64)
    u = _c(u, np.float64)
    out = np.empty_like(u)
    lib.orc_constant_eval(_ptr(values), values.size, _ptr(u), _ptr(out), u.size)
    return out


def dyadic_index(u, cap: int) -> np.ndarray:
    u = _c(u, np.float64)
    out = np.empty(u.shape, dtype=np.int64)
    lib.orc_dyadic_index(_ptr(u), cap, _ptr(out), u.size)
    return out


def dyadic_index32(u, cap: int) -> np.ndarray:
    u = _c(u, np.float32)
    out = np.empty(u.shape, dtype=np.int64)
    lib.orc_dyadic_index32(_ptr(u), cap, _ptr(out), u.size)
    return out


def dyadic_eval(coeffs, u) -> np.ndarray:
    coeffs = _c(coeffs, np.float64)
    u = _c(u, np.float64)
    out = np.empty_like(u)
    lib.orc_dyadic_eval(_ptr(coeffs), coeffs.shape[0] - 1, coeffs.shape[1], _ptr(u), _ptr(out), u.size)
    return out


def dyadic_eval32(coeffs32, u) -> np.ndarray:
    coeffs32 = _c(coeffs32, np.float32)
    u = _c(u, np.float32)
    out = np.empty_like(u)
    lib.orc_dyadic_eval32(_ptr(coeffs32), coeffs32.shape[0] - 1, coeffs32.shape[1], _ptr(u), _ptr(out),
                          u.size)
    return out


def ncchi2_eval(stacks, nu: float, u, lam) -> np.ndarray:
    stacks = _c(stacks, np.float64)
    u = _c(u, np.float64)
    lam = _c(np.atleast_1d(lam), np.float64)
    out = np.empty_like(u)
    _, n_knots, m1, k1 = stacks.shape
    lib.orc_ncchi2_eval(_ptr(stacks), n_knots, m1 - 1, k1, float(nu), _ptr(u), _ptr(lam), lam.size,
                        _ptr(out), u.size)
    return out


def subdyadic_eval32(coeffs, sub_bits: int, u) -> np.ndarray:
    """coeffs: f32 (degree+1, K, 2^sub_bits) natural layout (see oracle.c)."""
    coeffs = _c(coeffs, np.float32)
    u = _c(u, np.float32)
    out = np.empty_like(u)
    m1, K, nsub = coeffs.shape
    assert nsub == 1 << sub_bits
    lib.orc_subdyadic_eval32(_ptr(coeffs), m1 - 1, K, sub_bits, _ptr(u), _ptr(out), u.size)
    return out


def as241_f64(u) -> np.ndarray:
    u = _c(u, np.float64)
    out = np.empty_like(u)
    lib.orc_as241_f64(_ptr(u), _ptr(out), u.size)
    return out


def as241_f32(u) -> np.ndarray:
    u = _c(u, np.float32)
    out = np.empty_like(u)
    lib.orc_as241_f32(_ptr(u), _ptr(out), u.size)
    return out


# --------------------------------------------------------------------------
# Fused generators
# --------------------------------------------------------------------------

def pcg32_constant_f32(seed, seq, offset, values, n) -> np.ndarray:
    v32 = _c(values, np.float32)
    q = int(v32.size).bit_length() - 1
    out = np.empty(n, dtype=np.float32)
    lib.orc_pcg32_constant_f32(seed, seq, offset, _ptr(v32), q, _ptr(out), n)
    return out


def pcg32_subdyadic_f32(seed, seq, offset, coeffs, sub_bits, n) -> np.ndarray:
    coeffs = _c(coeffs, np.float32)
    m1, K, _ = coeffs.shape
    out = np.empty(n, dtype=np.float32)
    lib.orc_pcg32_subdyadic_f32(seed, seq, offset, _ptr(coeffs), m1 - 1, K, sub_bits, _ptr(out), n)
    return out


def pcg32_dyadic_f32(seed, seq, offset, coeffs32, n) -> np.ndarray:
    coeffs32 = _c(coeffs32, np.float32)
    out = np.empty(n, dtype=np.float32)
    lib.orc_pcg32_dyadic_f32(seed, seq, offset, _ptr(coeffs32), coeffs32.shape[0] - 1, coeffs32.shape[1],
                             _ptr(out), n)
    return out


def pcg32_as241_f64(seed, seq, offset, n) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib.orc_pcg32_as241_f64(seed, seq, offset, _ptr(out), n)
    return out


def pcg32_as241_f32(seed, seq, offset, n) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    lib.orc_pcg32_as241_f32(seed, seq, offset, _ptr(out), n)
    return out


# --------------------------------------------------------------------------
# MLMC path restatements (mlmc.py:164-331)
# --------------------------------------------------------------------------

def gbm_paths(*, mu, sigma, x0, t_end, level, n0, milstein, payoff_call, strike, coeffs,
              seed, seq, n_paths, path_lo=0, path_hi=None):
    """Per-path (p_fine_exact, p_coarse_exact, p_fine_approx, p_coarse_approx)."""
    path_hi = n_paths if path_hi is None else path_hi
    coeffs = _c(coeffs, np.float64)
    m = path_hi - path_lo
    outs = [np.empty(m) for _ in range(4)]
    lib.orc_gbm_paths(mu, sigma, x0, t_end, level, n0, int(milstein), int(payoff_call), strike,
                      _ptr(coeffs), coeffs.shape[0] - 1, coeffs.shape[1], seed, seq, n_paths,
                      path_lo, path_hi, *[_ptr(o) for o in outs])
    return tuple(outs)


def cir_euler_paths(*, kappa, theta, sigma, x0, t_end, level, n0, payoff_call, strike, coeffs,
                    seed, seq, n_paths, path_lo=0, path_hi=None, milstein=False):
    """CIR truncated Euler (mlmc.py:289-331) or, milstein=True, the truncated
    Milstein restatement (orc_cir_paths in oracle.c; no reference scheme)."""
    path_hi = n_paths if path_hi is None else path_hi
    coeffs = _c(coeffs, np.float64)
    m = path_hi - path_lo
    outs = [np.empty(m) for _ in range(4)]
    lib.orc_cir_paths(kappa, theta, sigma, x0, t_end, level, n0, int(milstein), int(payoff_call), strike,
                      _ptr(coeffs), coeffs.shape[0] - 1, coeffs.shape[1], seed, seq, n_paths,
                      path_lo, path_hi, *[_ptr(o) for o in outs])
    return tuple(outs)


def load_ref_kernels():
    """The reference's own compiled ``_kernels`` module from oracle/_ref, or None."""
    hits = glob.glob(os.path.join(_HERE, "_ref", "_kernels*.so"))
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_kernels", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod

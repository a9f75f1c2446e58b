"""ctypes binding of libarv_b200.so (the C ABI in include/approxrv_b200.h).

There is no fallback: if the library is missing or fails to load, importing
this module raises.  ``call(name, *args)`` invokes an entry point and turns a
non-zero status into the reference exception hierarchy (errors.py).
"""

from __future__ import annotations

import ctypes as C
import os

from . import _build
from .errors import raise_for

_u64, _i64, _int, _dbl, _p = C.c_uint64, C.c_int64, C.c_int, C.c_double, C.c_void_p


class LevelSpec(C.Structure):
    """arv_level_spec (include/approxrv_b200.h)."""

    _fields_ = [
        ("a", _dbl), ("b", _dbl), ("c", _dbl),
        ("x0", _dbl), ("t_end", _dbl),
        ("level", _int), ("n0", _int), ("scheme", _int), ("payoff", _int),
        ("strike", _dbl),
        ("seed", _u64), ("stream_id", _u64),
        ("n_paths_total", _i64), ("path_lo", _i64), ("path_count", _i64),
        ("rng", _int),
        ("sides", _int),
    ]


SCHEME_EM, SCHEME_MILSTEIN, SCHEME_CIR_EXACT, SCHEME_CIR_EULER_TRUNCATED, SCHEME_CIR_MILSTEIN_TRUNCATED = range(5)
PAYOFF_IDENTITY, PAYOFF_CALL = 0, 1
RNG_PCG32, RNG_PHILOX = 0, 1
SIDES_BOTH, SIDES_EXACT, SIDES_APPROX = 0, 1, 2
PHILOX_UNIFORM, PHILOX_CONSTANT, PHILOX_DYADIC, PHILOX_GAUSSIAN = range(4)

_SIGNATURES = {
    "arv_abi_version": ([], _int),
    "arv_last_error": ([], C.c_char_p),
    "arv_source_hash": ([], C.c_char_p),
    "arv_launch_count": ([], _u64),
    "arv_constant_eval": ([_p, _i64, _p, _p, _i64, _p], _int),
    "arv_dyadic_index": ([_p, _i64, _i64, _p, _p], _int),
    "arv_dyadic_index32": ([_p, _i64, _i64, _p, _p], _int),
    "arv_dyadic_eval": ([_p, _int, _i64, _p, _p, _i64, _p], _int),
    "arv_dyadic_eval32": ([_p, _int, _i64, _p, _p, _i64, _p], _int),
    "arv_ncchi2_eval": ([_p, _i64, _int, _i64, _dbl, _p, _p, _i64, _p, _i64, _p], _int),
    "arv_subdyadic_eval32": ([_p, _int, _int, _int, _p, _p, _i64, _p], _int),
    # host-buffer (numpy) convention: u / lam / out are host pointers
    "arv_host_constant_eval": ([_p, _i64, _p, _p, _i64, _p], _int),
    "arv_host_dyadic_index": ([_p, _i64, _i64, _p, _p], _int),
    "arv_host_dyadic_index32": ([_p, _i64, _i64, _p, _p], _int),
    "arv_host_dyadic_eval": ([_p, _int, _i64, _p, _p, _i64, _p], _int),
    "arv_host_dyadic_eval32": ([_p, _int, _i64, _p, _p, _i64, _p], _int),
    "arv_host_subdyadic_eval32": ([_p, _int, _int, _int, _p, _p, _i64, _p], _int),
    "arv_host_ncchi2_eval": ([_p, _i64, _int, _i64, _dbl, _p, _p, _i64, _p, _i64, _p], _int),
    "arv_host_gaussian_inv_cdf": ([_p, _p, _i64, _p], _int),
    "arv_gaussian_inv_cdf": ([_p, _p, _i64, _p], _int),
    "arv_gaussian_inv_cdf32": ([_p, _p, _i64, _p], _int),
    "arv_pcg32_words": ([_u64, _u64, _u64, _p, _i64, _p], _int),
    "arv_pcg32_uniform_f32": ([_u64, _u64, _u64, _p, _i64, _p], _int),
    "arv_pcg32_constant_f32": ([_u64, _u64, _u64, _p, _int, _p, _i64, _p], _int),
    "arv_pcg32_subdyadic_f32": ([_u64, _u64, _u64, _p, _int, _int, _int, _p, _i64, _p], _int),
    "arv_lattice_subdyadic_f32": ([_p, _int, _int, _int, _int, _p, _p, _p], _int),
    "arv_pcg32_gaussian_f64": ([_u64, _u64, _u64, _p, _i64, _p], _int),
    "arv_pcg32_gaussian_f32": ([_u64, _u64, _u64, _p, _i64, _p], _int),
    "arv_philox_words": ([_u64, _u64, _u64, _p, _i64, _p], _int),
    "arv_philox_eval_f64": ([_u64, _u64, _u64, _int, _p, _int, _i64, _p, _i64, _p], _int),
    "arv_store_probe": ([_p, _i64, _p], _int),
    "arv_store_probe_ex": ([_p, _i64, _int, _p], _int),
    "arv_set_tuning": ([_int, _int], _int),
    "arv_mlmc_workspace_bytes": ([_i64], _i64),
    "arv_mlmc_cir_workspace_bytes": ([_i64], _i64),
    "arv_mlmc_gaussian_level": ([C.POINTER(LevelSpec), _p, _int, _i64, _p, _p, _p, _i64, _p], _int),
    "arv_mlmc_cir_exact_level": ([C.POINTER(LevelSpec), _p, _i64, _int, _i64, _dbl, _p, _p, _p, _p, _i64, _p], _int),
    "arv_ncchi2_inv_cdf": ([_p, _p, _i64, _dbl, _p, _p, _p, _i64, _p], _int),
    "arv_ncchi2_inv_cdf_tol": ([_p, _p, _i64, _dbl, _p, _dbl, _p, _p, _i64, _p], _int),
    "arv_ncchi2_cdf": ([_p, _p, _i64, _dbl, _p, _i64, _p], _int),
    "arv_nc_certified_count": ([_p], _int),
    "arv_test_level_normals": ([_p, _p, _i64, _p], _int),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def _load() -> C.CDLL:
    # ARV_LIB_PATH: an alternative build of the same library (tuning experiments only)
    alt = os.environ.get("ARV_LIB_PATH")
    path = alt or _build.LIB_PATH
    if not alt:
        stale = _build.needs_build()
        if stale:
            # a library built from other sources must never load silently
            if os.environ.get("ARV_NO_AUTOBUILD"):
                raise ImportError(f"{path} is missing or was built from other sources; "
                                  "run `python -m paper_2012_09715_b200._build`")
            _build.build()
    lib = C.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError = stale or broken library: fail loudly
        fn.argtypes = args
        fn.restype = res
    if lib.arv_abi_version() != 1:
        raise ImportError("libarv_b200.so ABI version mismatch")
    return lib


lib = _load()
LIB_PATH = os.environ.get("ARV_LIB_PATH") or _build.LIB_PATH


_fns: dict = {}


def call(name: str, *args) -> None:
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(lib, name)
    rc = fn(*args)
    if rc:
        msg = lib.arv_last_error()
        raise_for(rc, (msg.decode() if msg else name) or name)


def launch_count() -> int:
    return int(lib.arv_launch_count())

"""Hot-path evaluation: uniforms in, approximate random variables out.

Mirrors the reference sampler API (approxrv/sampler.py:91-223): the eval
wrappers keep their names, argument meaning and errors, and route through
the drop-in kernel plugin (``_kernels``) on the device.  Inputs may be host
scalars/arrays (results come back to the host, like the reference) or CUDA
tensors (results stay on the device).

The uniform source is :class:`Pcg32Stream` (BASELINE.json: PCG32, seed 42,
stream 0), a counter-addressable stream like the reference's
``UniformStream`` (sampler.py:26-66): output ``i`` of ``(seed, stream_id)``
is fixed, ``counter`` advances by the words drawn, and any range can be
produced independently -- which is how samples shard across GPUs.  Its
``sample`` method is the fused generator: PCG32 -> table -> 128-bit stores,
with no input traffic at all.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _kernels as kernels
from ._native import call
from .errors import ConfigError, DomainError
from .tables import ConstantTable, DyadicPolyTable, NcChi2Table, SubDyadicTable

_MAX64 = (1 << 64) - 1


# ---------------------------------------------------------------------------
# Reference eval wrappers (sampler.py:91-206)
# ---------------------------------------------------------------------------

def _as_batch(u, dtype=torch.float64):
    """(batch, scalar?, host?) -- sampler.py:91-94.

    Host input stays a host array (the reference's f64 coercion and shape),
    and the plugin call runs the host-buffer pipeline; a CUDA tensor stays on
    the device (zero copy).
    """
    if dev.is_device_tensor(u):
        return dev.to_device(u.reshape(-1) if u.dim() else u.reshape(1), dtype, u.device), u.dim() == 0, False
    arr = np.asarray(u, dtype=np.float64)
    scalar = arr.ndim == 0
    return np.ascontiguousarray(np.atleast_1d(arr)), scalar, True


def _result(t, scalar: bool, host: bool, out=None):
    if out is not None and out is not t:
        dev.copy_out(out, t)
        return float(t.reshape(-1)[0]) if scalar else out
    if scalar:
        return float(t.reshape(-1)[0])
    return t


def _empty(ud, out, dtype=None):
    """The reference's `out = np.empty_like(arr)` (or the device twin)."""
    if isinstance(ud, np.ndarray):
        if isinstance(out, np.ndarray):
            return out
        return np.empty(ud.shape, dtype or ud.dtype)
    return torch.empty_like(ud)


def _coeffs(table, attr):
    return getattr(table, attr)


def eval_constant(table, u, out=None):
    """values[floor(2^q u)] per element (sampler.py:97-108)."""
    ud, scalar, host = _as_batch(u)
    od = _empty(ud, out)
    kernels.constant_eval(table.values, ud, od)
    return _result(od, scalar, host, out)


def dyadic_index(u, n_intervals: int = 1 << 62, dtype=np.float64):
    """Capped dyadic interval index from the float's exponent bits (sampler.py:111-124)."""
    ud, scalar, host = _as_batch(u)
    if dtype == np.float32:
        idx = kernels.dyadic_index32(ud if not host else np.ascontiguousarray(ud, dtype=np.float32), n_intervals)
    else:
        idx = kernels.dyadic_index(ud, n_intervals)
    if scalar:
        return int(idx.reshape(-1)[0])
    return idx.reshape(ud.shape) if host else idx


def _eval_general_decay(table, ud: torch.Tensor) -> torch.Tensor:
    """Analysis path for decay != 1/2 (sampler.py:127-141), as device tensor ops."""
    pred = ud < 0.5
    v = torch.where(pred, ud, 1.0 - ud)
    t = torch.log(2.0 * v) / math.log(table.decay)
    idx = torch.clamp(torch.ceil(t).to(torch.int64), 0, table.n_intervals)
    c = dev.table_on_device(table.coeffs, torch.float64, ud.device)
    acc = c[-1][idx]
    for row in range(c.shape[0] - 2, -1, -1):
        acc = acc * v + c[row][idx]
    return torch.where(pred, acc, -acc)


def eval_dyadic(table, u, dtype=np.float64, out=None):
    """Reflect-about-1/2, exponent-indexed Horner evaluation (sampler.py:144-172)."""
    if isinstance(table, SubDyadicTable):
        return eval_subdyadic(table, u, out=out)
    if getattr(table, "decay", 0.5) != 0.5:
        if dtype == np.float32:
            raise ConfigError("the float32 fast path requires decay rate 1/2")
        ud, scalar, host = _as_batch(u)
        res = _eval_general_decay(table, dev.to_device(ud, torch.float64) if host else ud)
        return _result(res.cpu().numpy().reshape(ud.shape) if host else res, scalar, host, out)
    ud, scalar, host = _as_batch(u)
    if dtype == np.float32:
        if host:
            ud = np.ascontiguousarray(ud, dtype=np.float32)
        else:
            ud = ud.to(torch.float32)
        od = _empty(ud, out)
        kernels.dyadic_eval32(table.coeffs32, ud, od)
    else:
        od = _empty(ud, out)
        kernels.dyadic_eval(table.coeffs, ud, od)
    return _result(od, scalar, host, out)


def eval_subdyadic(table: SubDyadicTable, u, out=None):
    """Octave x sub-interval table, float32 arithmetic (BASELINE.json config 2)."""
    ud, scalar, host = _as_batch(u)
    ud = np.ascontiguousarray(ud, dtype=np.float32) if host else ud.to(torch.float32)
    od = _empty(ud, out)
    kernels.subdyadic_eval32(table.coeffs32, table.sub_bits, ud, od)
    return _result(od, scalar, host, out)


def eval_ncchi2(table, u, lam, out=None):
    """Approximate non-central chi-squared quantiles (sampler.py:175-193)."""
    ud, scalar, host = _as_batch(u)
    if dev.is_device_tensor(lam):
        ld = lam.to(device=lam.device, dtype=torch.float64)
        if bool((ld < 0.0).any()):
            raise DomainError("lambda must be >= 0")
        lam_shape = tuple(ld.shape)
        if host:
            ud = dev.to_device(ud, torch.float64, ld.device)
            host = False
    else:
        lam_arr = np.asarray(lam, dtype=np.float64)
        if np.any(lam_arr < 0.0):
            raise DomainError("lambda must be >= 0")
        lam_shape = lam_arr.shape
        ld = np.ascontiguousarray(lam_arr.reshape(-1)) if host else \
            dev.to_device(lam_arr.reshape(-1), torch.float64, ud.device)
    if len(lam_shape) == 0:
        ld = ld.reshape(1)
    elif tuple(lam_shape) != tuple(ud.shape):
        raise ConfigError("per-element lambda must match the shape of u")
    od = _empty(ud, out)
    kernels.ncchi2_eval(table.eval_stacks, table.nu, ud, ld.reshape(-1), od)
    return _result(od, scalar, host, out)


def evaluate(table, u, lam=None, dtype=np.float64, out=None):
    """Evaluate any table type on a batch of uniforms (sampler.py:196-206)."""
    if _is(table, "ConstantTable", ConstantTable):
        return eval_constant(table, u, out=out)
    if isinstance(table, SubDyadicTable):
        return eval_subdyadic(table, u, out=out)
    if _is(table, "DyadicPolyTable", DyadicPolyTable):
        return eval_dyadic(table, u, dtype=dtype, out=out)
    if _is(table, "NcChi2Table", NcChi2Table):
        if lam is None:
            raise ConfigError("non-central chi-squared tables need lam")
        return eval_ncchi2(table, u, lam, out=out)
    raise ConfigError(f"cannot evaluate object of type {type(table).__name__}")


def _is(obj, name, cls) -> bool:
    """isinstance, also accepting the reference's own table classes by name."""
    return isinstance(obj, cls) or type(obj).__name__ == name


def gaussian_inv_cdf(u, out=None):
    """Exact AS241 quantile on the device (exact_dist.py:87-126), validating u."""
    ud, scalar, host = _as_batch(u)
    if host:
        bad = ud.size and bool(np.any(~np.isfinite(ud) | (ud <= 0.0) | (ud >= 1.0)))
    else:
        bad = ud.numel() and bool(((~torch.isfinite(ud)) | (ud <= 0.0) | (ud >= 1.0)).any())
    if bad:
        raise DomainError("gaussian_inv_cdf requires 0 < u < 1")
    od = _empty(ud, out)
    kernels.gaussian_inv_cdf(ud, od)
    return _result(od, scalar, host, out)


# ---------------------------------------------------------------------------
# PCG32 stream and fused generators
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class GaussianSamplePair:
    """Exact and approximate Gaussian samples from one shared uniform (sampler.py:69-74)."""

    z_exact: float
    z_approx: float


@dataclass(frozen=True)
class CoupledGaussianBatch:
    """Arrays of coupled samples; pair i derives from the same uniform (sampler.py:77-88)."""

    z_exact: object
    z_approx: object

    def __len__(self) -> int:
        return int(self.z_exact.shape[0])

    def __getitem__(self, i) -> GaussianSamplePair:
        return GaussianSamplePair(float(self.z_exact[i]), float(self.z_approx[i]))


@dataclass
class Pcg32Stream:
    """Counter-addressable PCG32 stream on the device (the UniformStream analogue).

    ``(seed, stream_id)`` = PCG32 ``(initstate, initseq)``; ``counter`` is the
    index of the next 32-bit output.  f32 uniforms are ((w >> 9) + 0.5) 2^-23
    (exact, open interval, never 1/2); f64 uniforms are (w + 0.5) 2^-32.
    """

    seed: int = 42
    stream_id: int = 0
    counter: int = 0

    def __post_init__(self):
        if not (0 <= int(self.seed) <= _MAX64 and 0 <= int(self.stream_id) < (1 << 63)):
            raise ConfigError("seed must fit in 64 bits and stream_id in 63 bits")
        if self.counter < 0:
            raise ConfigError("counter must be >= 0")

    # -- bookkeeping --------------------------------------------------------
    def _take(self, n: int) -> int:
        if n < 0:
            raise ConfigError("cannot draw a negative number of words")
        start = self.counter
        self.counter = start + n
        return start

    def child(self, stream_id: int) -> "Pcg32Stream":
        return Pcg32Stream(self.seed, stream_id)

    def _out(self, out, n, dtype, device):
        if out is None:
            return torch.empty(n, dtype=dtype, device=device or dev.require_cuda())
        if not (dev.is_device_tensor(out) and out.dtype == dtype and out.is_contiguous() and out.numel() == n):
            raise ConfigError(f"out must be a contiguous CUDA {dtype} tensor of {n} elements")
        return out

    # -- raw draws ----------------------------------------------------------
    def words(self, n: int, out=None, device=None) -> torch.Tensor:
        start = self._take(n)
        o = self._out(out, n, torch.uint32, device)
        call("arv_pcg32_words", self.seed, self.stream_id, start, o.data_ptr(), n, dev.stream_handle(o.device))
        return o

    def uniforms(self, n: int, dtype=np.float32, out=None, device=None) -> torch.Tensor:
        if dtype == np.float32:
            start = self._take(n)
            o = self._out(out, n, torch.float32, device)
            call("arv_pcg32_uniform_f32", self.seed, self.stream_id, start, o.data_ptr(), n,
                 dev.stream_handle(o.device))
            return o
        w = self.words(n, device=device)
        u = (w.to(torch.int64).to(torch.float64) + 0.5) * 2.0**-32
        if out is not None:
            out.copy_(u)
            return out
        return u

    # -- fused generators ---------------------------------------------------
    def sample(self, table, n: int, out=None, device=None) -> torch.Tensor:
        """n approximate Gaussian samples (f32) generated in one fused kernel.

        ``table`` is a ConstantTable, DyadicPolyTable (reference layout),
        SubDyadicTable, or the string ``"exact"`` (AS241 in f32 arithmetic).
        """
        o = self._out(out, n, torch.float32, device)
        s = dev.stream_handle(o.device)
        if _is(table, "ConstantTable", ConstantTable):
            vals = dev.table_on_device(_values32(table), torch.float32, o.device)
            q = int(vals.numel()).bit_length() - 1
            start = self._take(n)
            call("arv_pcg32_constant_f32", self.seed, self.stream_id, start, vals.data_ptr(), q, o.data_ptr(), n, s)
        elif isinstance(table, SubDyadicTable):
            c = dev.table_on_device(table.coeffs32, torch.float32, o.device)
            start = self._take(n)
            call("arv_pcg32_subdyadic_f32", self.seed, self.stream_id, start, c.data_ptr(), table.degree,
                 table.n_octaves, table.sub_bits, o.data_ptr(), n, s)
        elif _is(table, "DyadicPolyTable", DyadicPolyTable):
            if getattr(table, "decay", 0.5) != 0.5:
                raise ConfigError("the float32 fast path requires decay rate 1/2")
            nat = _natural32(table)
            c = dev.table_on_device(nat, torch.float32, o.device)
            start = self._take(n)
            call("arv_pcg32_subdyadic_f32", self.seed, self.stream_id, start, c.data_ptr(), table.degree,
                 table.n_intervals, 0, o.data_ptr(), n, s)
        elif table == "exact":
            start = self._take(n)
            call("arv_pcg32_gaussian_f32", self.seed, self.stream_id, start, o.data_ptr(), n, s)
        else:
            raise ConfigError(f"cannot sample from object of type {type(table).__name__}")
        return o

    def sample_exact64(self, n: int, out=None, device=None) -> torch.Tensor:
        """AS241 in f64 of the same f32-lattice uniforms (exact comparator)."""
        o = self._out(out, n, torch.float64, device)
        start = self._take(n)
        call("arv_pcg32_gaussian_f64", self.seed, self.stream_id, start, o.data_ptr(), n,
             dev.stream_handle(o.device))
        return o

    def sample_host(self, table, n: int, out=None, chunk: int = 1 << 25, sync: bool = True):
        """Fused generation straight into a host buffer (the end-to-end path).

        The batch is produced in chunks on the current stream while a side
        stream drains finished chunks device->host into ``out`` (a pinned
        CPU tensor for full PCIe rate; allocated pinned if None), so the
        HBM-side generation hides behind the host link.  Returns ``out``.
        """
        device = dev.require_cuda()
        if out is None:
            out = torch.empty(n, dtype=torch.float32, pin_memory=True)
        if not isinstance(out, torch.Tensor):
            host = np.asarray(out)
            # a non-contiguous or read-only array would be filled through a
            # temporary copy and the caller's buffer never written: refuse it
            if not (host.flags.c_contiguous and host.flags.writeable):
                raise ConfigError("out must be a C-contiguous, writeable float32 array")
            out = torch.from_numpy(host)
        if out.numel() != n or out.dtype != torch.float32 or out.is_cuda:
            raise ConfigError("out must be a host float32 buffer of n elements")
        chunk = max(4, min(chunk, n)) & ~3
        comp = torch.cuda.current_stream(device)
        copy = _side_stream(device)
        bufs = _chunk_buffers(device, chunk)
        freed = [None, None]
        start = self.counter
        for i, lo in enumerate(range(0, n, chunk)):
            hi = min(lo + chunk, n)
            b = bufs[i & 1]
            if freed[i & 1] is not None:
                comp.wait_event(freed[i & 1])
            self.counter = start + lo
            self.sample(table, hi - lo, out=b[: hi - lo])
            made = torch.cuda.Event()
            made.record(comp)
            copy.wait_event(made)
            with torch.cuda.stream(copy):
                out[lo:hi].copy_(b[: hi - lo], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            freed[i & 1] = ev
        self.counter = start + n
        comp.wait_stream(copy)
        if sync:
            comp.synchronize()
        return out


@dataclass
class PhiloxStream:
    """The reference's UniformStream (sampler.py:26-66), replayed on the device.

    Philox-4x64-10 keyed with (seed, stream_id); ``counter`` indexes 64-bit
    words; ``uniforms`` are ((w >> 11) + 0.5) 2^-53 in f64 -- bit-exact with
    ``approxrv.sampler.UniformStream(seed, stream_id, counter)``, so device
    results can be replayed path by path against the reference.
    """

    seed: int
    stream_id: int = 0
    counter: int = 0

    def __post_init__(self):
        if not 0 <= int(self.seed) <= _MAX64 or not 0 <= int(self.stream_id) <= _MAX64:
            raise ConfigError("seed and stream_id must fit in 64 bits")

    def _take(self, n: int) -> int:
        if n < 0:
            raise ConfigError("cannot draw a negative number of words")
        start = self.counter
        self.counter = start + n
        return start

    def child(self, stream_id: int) -> "PhiloxStream":
        return PhiloxStream(self.seed, stream_id)

    def raw_words(self, n: int, device=None) -> torch.Tensor:
        """The next n raw 64-bit words (uint64 device tensor), advancing the counter."""
        start = self._take(n)
        o = torch.empty(n, dtype=torch.uint64, device=device or dev.require_cuda())
        call("arv_philox_words", self.seed, self.stream_id, start, o.data_ptr(), n, dev.stream_handle(o.device))
        return o

    def _eval(self, kind, n, table=None, degree=0, cols=0, out=None, device=None):
        start = self._take(n)
        o = out if out is not None else torch.empty(n, dtype=torch.float64, device=device or dev.require_cuda())
        if not (dev.is_device_tensor(o) and o.dtype == torch.float64 and o.is_contiguous() and o.numel() == n):
            raise ConfigError(f"out must be a contiguous CUDA float64 tensor of {n} elements")
        tp = table.data_ptr() if table is not None else None
        call("arv_philox_eval_f64", self.seed, self.stream_id, start, kind, tp, degree, cols, o.data_ptr(), n,
             dev.stream_handle(o.device))
        return o

    def uniforms(self, n: int, out=None, device=None) -> torch.Tensor:
        """n doubles in (0, 1) (sampler.py:59-62)."""
        return self._eval(_PH_UNIFORM, n, out=out, device=device)

    def sample(self, table, n: int, out=None, device=None) -> torch.Tensor:
        """Fused ``evaluate(table, self.uniforms(n))`` in f64 (the reference default).

        ``table`` is a ConstantTable, DyadicPolyTable (decay 1/2) or ``"exact"`` (AS241).
        """
        device = device or dev.require_cuda()
        if _is(table, "ConstantTable", ConstantTable):
            v = dev.table_on_device(table.values, torch.float64, device)
            return self._eval(_PH_CONSTANT, n, v, 0, v.numel(), out, device)
        if _is(table, "DyadicPolyTable", DyadicPolyTable):
            if getattr(table, "decay", 0.5) != 0.5:
                raise ConfigError("the fused path requires decay rate 1/2")
            c = dev.table_on_device(table.coeffs, torch.float64, device)
            return self._eval(_PH_DYADIC, n, c, c.shape[0] - 1, c.shape[1], out, device)
        if isinstance(table, str) and table == "exact":
            return self._eval(_PH_GAUSSIAN, n, out=out, device=device)
        raise ConfigError(f"cannot sample from object of type {type(table).__name__}")


_PH_UNIFORM, _PH_CONSTANT, _PH_DYADIC, _PH_GAUSSIAN = range(4)

_SIDE: dict = {}
_BUFS: dict = {}


def _side_stream(device) -> torch.cuda.Stream:
    s = _SIDE.get(device.index)
    if s is None:
        s = _SIDE[device.index] = torch.cuda.Stream(device)
    return s


def _chunk_buffers(device, chunk: int):
    key = (device.index, chunk)
    b = _BUFS.get(key)
    if b is None:
        b = _BUFS[key] = [torch.empty(chunk, dtype=torch.float32, device=device) for _ in range(2)]
    return b


def _values32(table) -> np.ndarray:
    v = getattr(table, "values32", None)
    if v is None:
        v = np.asarray(table.values, dtype=np.float32)
        v.setflags(write=False)
    return v


_NAT_CACHE: dict = {}


def _natural32(table) -> np.ndarray:
    nat = getattr(table, "natural32", None)
    if nat is not None:
        return nat
    key = id(table)
    hit = _NAT_CACHE.get(key)
    if hit is None or hit[0] is not table:
        arr = np.ascontiguousarray(np.asarray(table.coeffs, dtype=np.float32)[:, 1:, None])
        arr.setflags(write=False)
        hit = (table, arr)
        _NAT_CACHE[key] = hit
    return hit[1]


def sample_coupled(stream, table, n: int) -> CoupledGaussianBatch:
    """Draw n uniforms once; exact and approximate Gaussians (sampler.py:209-218).

    ``stream`` is a Pcg32Stream (f64 uniforms (w + 0.5) 2^-32) or a
    PhiloxStream (the reference's own UniformStream uniforms, so the pair
    matches the reference's sample_coupled bit for bit on the table side).
    """
    u = stream.uniforms(n) if isinstance(stream, PhiloxStream) else stream.uniforms(n, dtype=np.float64)
    z_exact = torch.empty_like(u)
    kernels.gaussian_inv_cdf(u, z_exact)
    z_approx = evaluate(table, u)
    if isinstance(z_approx, torch.Tensor) and z_approx.dtype != torch.float64:
        z_approx = z_approx.to(torch.float64)
    return CoupledGaussianBatch(z_exact=z_exact, z_approx=z_approx)


def gaussian_exact_batch(u):
    """Exact quantile of a uniform batch (sampler.py:221-223): AS241 on the device."""
    return gaussian_inv_cdf(u)


# The reference's name for its Philox-4x64-10 stream (sampler.py:26-66).
UniformStream = PhiloxStream


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of ``n_total`` samples owned by ``rank``.

    Boundaries are multiples of 8 samples (32 bytes), so a shard written into
    a slice of a shared buffer keeps the 256-bit store path."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError("bad rank/world")
    groups = (n_total + 7) // 8
    per = groups // world
    extra = groups % world
    g_lo = rank * per + min(rank, extra)
    g_hi = g_lo + per + (1 if rank < extra else 0)
    return min(8 * g_lo, n_total), min(8 * g_hi, n_total)

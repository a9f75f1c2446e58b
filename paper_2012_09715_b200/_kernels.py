"""Drop-in replacement of the reference kernel plugin ``approxrv._kernels``.

Same six functions, same argument order and meaning, same results as the
Cython module (``_kernels.pyx:16-143``), executed by hand-written sm_100a
kernels through the C ABI of libarv_b200.so.  ``COMPILED`` is True, as for the
reference's compiled backend (``_backend.py:27-29``).

Arguments may be numpy arrays (the reference's calling convention) or CUDA
torch tensors (zero-copy; results stay on the device, ordered on torch's
current stream).  Host arrays go through the library's host-buffer entry
points (``arv_host_*``, csrc/arv_host.cu): chunks are staged through pinned
buffers with the host copies, H2D, kernel and D2H overlapped, and the
caller's ``out`` is written once, in place, before the call returns.  As in
the reference, ``out`` is caller-allocated and the index functions return a
new int64 array.  Kernels do not validate ``u``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dev
from ._native import call

COMPILED = True


_NP = {torch.float64: np.float64, torch.float32: np.float32, torch.int64: np.int64}


def _host(*arrays) -> bool:
    """True when no argument is a CUDA tensor: the numpy (host) convention."""
    return not any(isinstance(a, torch.Tensor) for a in arrays)


def _host_in(x, dtype: torch.dtype) -> np.ndarray:
    """1-D C-contiguous host array of the kernel's dtype (copied only if needed)."""
    return np.ascontiguousarray(np.asarray(x, dtype=_NP[dtype]).reshape(-1))


def _host_out(out, dtype: torch.dtype, n: int):
    """(host buffer the kernel writes, whether it must be copied into ``out``)."""
    nd = _NP[dtype]
    if isinstance(out, np.ndarray) and out.dtype == nd and out.flags.c_contiguous and out.flags.writeable \
            and out.size == n:
        return out.reshape(-1), False
    return np.empty(n, nd), True


def _host_finish(out, buf, copy_back: bool) -> None:
    if copy_back:
        np.copyto(out, buf.reshape(np.shape(out)), casting="unsafe")


def _dev_out(out, like: torch.Tensor, dtype: torch.dtype):
    """(device tensor to write, needs_copy_back)."""
    if isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == dtype and out.is_contiguous() \
            and out.numel() == like.numel():
        return out, False
    return torch.empty(like.shape, dtype=dtype, device=like.device), True


def _finish(out, t: torch.Tensor, copy_back: bool) -> None:
    if copy_back:
        dev.copy_out(out, t)


def constant_eval(values, u, out) -> None:
    """_kernels.pyx:16-23: out[i] = values[min(int(nvals * u[i]), nvals - 1)]."""
    if _host(u, out):
        uh = _host_in(u, torch.float64)
        vd = dev.table_on_device(values, torch.float64)
        oh, back = _host_out(out, torch.float64, uh.size)
        call("arv_host_constant_eval", vd.data_ptr(), vd.numel(), uh.ctypes.data, oh.ctypes.data, uh.size,
             dev.stream_handle(vd.device))
        return _host_finish(out, oh, back)
    ud = dev.to_device(u, torch.float64)
    vd = dev.table_on_device(values, torch.float64, ud.device)
    od, back = _dev_out(out, ud, torch.float64)
    call("arv_constant_eval", vd.data_ptr(), vd.numel(), ud.data_ptr(), od.data_ptr(), ud.numel(),
         dev.stream_handle(ud.device))
    _finish(out, od, back)


def _index(name, u, cap, dtype):
    if _host(u):
        uh = _host_in(u, dtype)
        oh = np.empty(uh.size, np.int64)
        call(name.replace("arv_", "arv_host_"), uh.ctypes.data, uh.size, int(cap), oh.ctypes.data,
             dev.stream_handle(dev.require_cuda()))
        return oh
    ud = dev.to_device(u, dtype)
    od = torch.empty(ud.shape, dtype=torch.int64, device=ud.device)
    call(name, ud.data_ptr(), ud.numel(), int(cap), od.data_ptr(), dev.stream_handle(ud.device))
    if dev.is_device_tensor(u):
        return od
    return od.cpu().numpy()


def dyadic_index(u, cap):
    """_kernels.pyx:26-38: 1022 - (bits(u) >> 52), capped at ``cap``."""
    return _index("arv_dyadic_index", u, cap, torch.float64)


def dyadic_index32(u, cap):
    """_kernels.pyx:41-53: 126 - (bits(u) >> 23), capped at ``cap``."""
    return _index("arv_dyadic_index32", u, cap, torch.float32)


def _dyadic(name, coeffs, u, out, dtype):
    if _host(u, out):
        uh = _host_in(u, dtype)
        cd = dev.table_on_device(coeffs, dtype)
        if cd.dim() != 2:
            raise ValueError("coeffs must be (degree+1, K+1)")
        oh, back = _host_out(out, dtype, uh.size)
        call(name.replace("arv_", "arv_host_"), cd.data_ptr(), cd.shape[0] - 1, cd.shape[1], uh.ctypes.data,
             oh.ctypes.data, uh.size, dev.stream_handle(cd.device))
        return _host_finish(out, oh, back)
    ud = dev.to_device(u, dtype)
    cd = dev.table_on_device(coeffs, dtype, ud.device)
    if cd.dim() != 2:
        raise ValueError("coeffs must be (degree+1, K+1)")
    od, back = _dev_out(out, ud, dtype)
    call(name, cd.data_ptr(), cd.shape[0] - 1, cd.shape[1], ud.data_ptr(), od.data_ptr(), ud.numel(),
         dev.stream_handle(ud.device))
    _finish(out, od, back)


def dyadic_eval(coeffs, u, out) -> None:
    """_kernels.pyx:56-73 (float64)."""
    _dyadic("arv_dyadic_eval", coeffs, u, out, torch.float64)


def dyadic_eval32(coeffs, u, out) -> None:
    """_kernels.pyx:76-93 (float32 input, coefficients and arithmetic)."""
    _dyadic("arv_dyadic_eval32", coeffs, u, out, torch.float32)


def ncchi2_eval(stacks, nu, u, lam, out) -> None:
    """_kernels.pyx:96-143: interpolated non-central chi-squared table."""
    if _host(u, lam, out):
        uh = _host_in(u, torch.float64)
        lh = _host_in(lam, torch.float64)
        sd = dev.table_on_device(stacks, torch.float64)
        if sd.dim() != 4 or sd.shape[0] != 2:
            raise ValueError("stacks must be (2, n_knots, degree+1, K+1)")
        oh, back = _host_out(out, torch.float64, uh.size)
        call("arv_host_ncchi2_eval", sd.data_ptr(), sd.shape[1], sd.shape[2] - 1, sd.shape[3], float(nu),
             uh.ctypes.data, lh.ctypes.data, lh.size, oh.ctypes.data, uh.size, dev.stream_handle(sd.device))
        return _host_finish(out, oh, back)
    ud = dev.to_device(u, torch.float64)
    sd = dev.table_on_device(stacks, torch.float64, ud.device)
    ld = dev.to_device(lam, torch.float64, ud.device).reshape(-1)
    if sd.dim() != 4 or sd.shape[0] != 2:
        raise ValueError("stacks must be (2, n_knots, degree+1, K+1)")
    od, back = _dev_out(out, ud, torch.float64)
    call("arv_ncchi2_eval", sd.data_ptr(), sd.shape[1], sd.shape[2] - 1, sd.shape[3], float(nu), ud.data_ptr(),
         ld.data_ptr(), ld.numel(), od.data_ptr(), ud.numel(), dev.stream_handle(ud.device))
    _finish(out, od, back)


# ---------------------------------------------------------------------------
# Extensions beyond the reference plugin (same calling convention).
# ---------------------------------------------------------------------------

def subdyadic_eval32(coeffs, sub_bits: int, u, out) -> None:
    """Octave x sub-interval f32 table, coeffs (degree+1, K, 2^sub_bits)."""
    if _host(u, out):
        uh = _host_in(u, torch.float32)
        cd = dev.table_on_device(coeffs, torch.float32)
        if cd.dim() != 3 or cd.shape[2] != 1 << sub_bits:
            raise ValueError("coeffs must be (degree+1, K, 2**sub_bits)")
        oh, back = _host_out(out, torch.float32, uh.size)
        call("arv_host_subdyadic_eval32", cd.data_ptr(), cd.shape[0] - 1, cd.shape[1], int(sub_bits),
             uh.ctypes.data, oh.ctypes.data, uh.size, dev.stream_handle(cd.device))
        return _host_finish(out, oh, back)
    ud = dev.to_device(u, torch.float32)
    cd = dev.table_on_device(coeffs, torch.float32, ud.device)
    if cd.dim() != 3 or cd.shape[2] != 1 << sub_bits:
        raise ValueError("coeffs must be (degree+1, K, 2**sub_bits)")
    od, back = _dev_out(out, ud, torch.float32)
    call("arv_subdyadic_eval32", cd.data_ptr(), cd.shape[0] - 1, cd.shape[1], int(sub_bits), ud.data_ptr(),
         od.data_ptr(), ud.numel(), dev.stream_handle(ud.device))
    _finish(out, od, back)


def gaussian_inv_cdf(u, out) -> None:
    """AS241 (exact_dist.py:87-126) in float64, without domain validation."""
    if _host(u, out):
        uh = _host_in(u, torch.float64)
        oh, back = _host_out(out, torch.float64, uh.size)
        call("arv_host_gaussian_inv_cdf", uh.ctypes.data, oh.ctypes.data, uh.size,
             dev.stream_handle(dev.require_cuda()))
        return _host_finish(out, oh, back)
    ud = dev.to_device(u, torch.float64)
    od, back = _dev_out(out, ud, torch.float64)
    call("arv_gaussian_inv_cdf", ud.data_ptr(), od.data_ptr(), ud.numel(), dev.stream_handle(ud.device))
    _finish(out, od, back)


def gaussian_inv_cdf32(u, out) -> None:
    """The AS241 rational evaluated in float32 arithmetic."""
    ud = dev.to_device(u, torch.float32)
    od, back = _dev_out(out, ud, torch.float32)
    call("arv_gaussian_inv_cdf32", ud.data_ptr(), od.data_ptr(), ud.numel(), dev.stream_handle(ud.device))
    _finish(out, od, back)


__all__ = [
    "COMPILED", "constant_eval", "dyadic_index", "dyadic_index32", "dyadic_eval", "dyadic_eval32",
    "ncchi2_eval", "subdyadic_eval32", "gaussian_inv_cdf", "gaussian_inv_cdf32",
]

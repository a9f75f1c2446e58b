"""Device plumbing: torch supplies memory and streams; the math is in libarv_b200.

* ``to_device(x, dtype)`` -- contiguous CUDA tensor view of a torch tensor or
  an H2D copy of a host array (the reference-facing, host-buffer path).
* ``table_on_device(arr, dtype)`` -- frozen reference tables (read-only
  numpy arrays, tables.py:19-24) are uploaded once per (buffer, dtype,
  device) and cached; they are immutable, so the cache never goes stale.
* ``stream_handle()`` -- the cudaStream_t of torch's current stream, passed
  to every C-ABI call so kernels order with the caller's torch work.
"""

from __future__ import annotations

import threading
from collections import OrderedDict

import numpy as np
import torch

from .errors import ConfigError, DeviceError

_NP_TO_TORCH = {
    np.dtype(np.float64): torch.float64,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.uint32): torch.uint32,
}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("approxrv-b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(device: torch.device | None = None) -> int:
    # torch's own fast accessor for the current cudaStream_t (~0.3 us against
    # ~2 us for current_stream().cuda_stream, which builds a Stream object)
    if _raw_stream is not None:
        idx = torch.cuda.current_device() if device is None or device.index is None else device.index
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def is_device_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device(x, dtype: torch.dtype, device: torch.device | None = None) -> torch.Tensor:
    """Contiguous CUDA tensor of ``dtype``; host inputs are copied (H2D)."""
    device = device or require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        if t.device != device or t.dtype != dtype:
            t = t.to(device=device, dtype=dtype, non_blocking=True)
        return t.contiguous()
    arr = np.asarray(x)
    tdt = _NP_TO_TORCH.get(arr.dtype)
    if tdt is None or tdt != dtype:
        arr = arr.astype(_torch_to_np(dtype))
    arr = np.ascontiguousarray(arr)
    if not arr.flags.writeable:
        arr = arr.copy()
    return torch.from_numpy(arr).to(device=device, non_blocking=False)


def _torch_to_np(dtype: torch.dtype):
    for k, v in _NP_TO_TORCH.items():
        if v == dtype:
            return k
    raise ConfigError(f"unsupported dtype {dtype}")


_TABLE_CACHE_MAX = 64  # device copies of distinct read-only tables kept (LRU)
_table_cache: "OrderedDict" = OrderedDict()
_table_lock = threading.Lock()


def table_on_device(arr, dtype: torch.dtype, device: torch.device | None = None) -> torch.Tensor:
    """Cached device copy of an immutable host table (keyed by buffer identity)."""
    if isinstance(arr, torch.Tensor) and arr.is_cuda:
        return to_device(arr, dtype, arr.device)
    device = device or require_cuda()
    a = np.asarray(arr)
    if a.flags.writeable:
        # Mutable host arrays cannot be cached safely; upload every call.
        return to_device(a, dtype, device)
    # keyed by object identity: the entry holds `a`, so its id cannot be reused
    # while cached, and read-only arrays never change
    key = (id(a), dtype, device.index)
    with _table_lock:
        hit = _table_cache.get(key)
        if hit is not None and hit[0] is a:
            _table_cache.move_to_end(key)
            return hit[1]
        t = to_device(a, dtype, device)
        _table_cache[key] = (a, t)  # holds `a`, so its buffer address cannot be reused while cached
        while len(_table_cache) > _TABLE_CACHE_MAX:
            _table_cache.popitem(last=False)
        return t


def copy_out(dst, src) -> None:
    """Write a result (device tensor or host array) into the caller's ``out``."""
    if isinstance(dst, torch.Tensor):
        if isinstance(src, np.ndarray):
            src = torch.from_numpy(np.ascontiguousarray(src))
        if dst.data_ptr() != src.data_ptr():
            dst.copy_(src.view(dst.shape) if src.numel() == dst.numel() else src)
        return
    host = src if isinstance(src, np.ndarray) else src.cpu().numpy()
    np.copyto(dst, host.reshape(np.shape(dst)), casting="unsafe")

"""Exact reference distributions on the device (mirrors approxrv/exact_dist.py).

* ``gaussian_inv_cdf(u)``          AS241 / PPND16 (exact_dist.py:87-126), device f64.
* ``ncchi2_cdf(x, nu, lam)``       Poisson mixture of regularized gammas
  (exact_dist.py:215-235) by the downward sweep of csrc/arv_ncchi2.cuh;
  within 2e-13 of scipy's CDFLIB ``chndtr`` (tests/test_gpu_mlmc.py).
* ``ncchi2_inv_cdf_batch(u, nu, lam, x0=None, tol=1e-9)``  the quantile
  (exact_dist.py:381-461): bisection-safeguarded Newton in the reference's
  bracket with its tol_f, one thread per element, scalar or per-element
  lambda; NumericalError when a residual |F(x) - u| exceeds 1e-8.
* ``cir_transition_params(x_prev, kappa, theta, sigma, dt)``  (exact_dist.py:
  542-567), host arithmetic.

Inputs may be numpy arrays (copied to the GPU, results returned as numpy,
the reference's convention) or CUDA tensors (results stay on the device).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _device as dev
from ._native import call
from .errors import DomainError, NumericalError
from .sampler import gaussian_inv_cdf  # noqa: F401  (re-exported under the reference's module)

__all__ = ["gaussian_inv_cdf", "ncchi2_cdf", "ncchi2_inv_cdf_batch", "cir_transition_params"]


def _validate(nu: float, lam) -> float:
    nu = float(nu)
    if not (math.isfinite(nu) and nu > 0.0):
        raise DomainError(f"degrees of freedom must be finite and > 0, got {nu}")
    return nu


def _back(t: torch.Tensor, like, scalar: bool):
    if dev.is_device_tensor(like):
        return t
    a = t.cpu().numpy()
    return float(a[0]) if scalar else a


def ncchi2_cdf(x, nu, lam):
    """CDF of the non-central chi-squared distribution (exact_dist.py:215-235)."""
    nu = _validate(nu, lam)
    lam = float(lam)
    if not (math.isfinite(lam) and lam >= 0.0):
        raise DomainError(f"non-centrality must be finite and >= 0, got {lam}")
    scalar = np.ndim(x) == 0 and not dev.is_device_tensor(x)
    xd = dev.to_device(np.atleast_1d(x) if scalar else x, torch.float64).reshape(-1)
    if xd.numel() and (not bool(torch.isfinite(xd).all()) or bool((xd < 0).any())):
        raise DomainError("ncchi2_cdf requires finite x >= 0")
    ld = torch.full((1,), lam, dtype=torch.float64, device=xd.device)
    out = torch.empty_like(xd)
    call("arv_ncchi2_cdf", xd.data_ptr(), ld.data_ptr(), 1, nu, out.data_ptr(), xd.numel(),
         dev.stream_handle(xd.device))
    out.clamp_(0.0, 1.0)
    return _back(out, x, scalar)


def ncchi2_inv_cdf_batch(u, nu, lam, x0=None, tol=1e-9):
    """Vectorized non-central chi-squared quantile (exact_dist.py:381-461)."""
    scalar = np.ndim(u) == 0 and not dev.is_device_tensor(u)
    ud = dev.to_device(np.atleast_1d(u) if scalar else u, torch.float64).reshape(-1)
    if ud.numel() and (bool((ud <= 0).any()) or bool((ud >= 1).any()) or not bool(torch.isfinite(ud).all())):
        raise DomainError("ncchi2_inv_cdf_batch requires 0 < u < 1")
    per_element = np.ndim(lam) > 0 or (dev.is_device_tensor(lam) and lam.dim() > 0)
    nu = _validate(nu, lam)
    ld = dev.to_device(np.atleast_1d(lam) if not per_element else lam, torch.float64, ud.device).reshape(-1)
    if not per_element:
        if not (math.isfinite(float(ld[0])) and float(ld[0]) >= 0.0):
            raise DomainError(f"non-centrality must be finite and >= 0, got {float(ld[0])}")
    elif bool((ld < 0).any()) or not bool(torch.isfinite(ld).all()):
        raise DomainError("invalid (nu, lambda) in batch quantile")
    if per_element and ld.numel() != ud.numel():
        ld = ld.expand(ud.numel()).contiguous() if ld.numel() == 1 else torch.broadcast_to(ld, ud.shape).contiguous()
    xd = None if x0 is None else dev.to_device(x0, torch.float64, ud.device).reshape(-1)
    out = torch.empty_like(ud)
    resid = torch.empty_like(ud)
    call("arv_ncchi2_inv_cdf_tol", ud.data_ptr(), ld.data_ptr(), ld.numel(), nu,
         xd.data_ptr() if xd is not None else None, float(tol), out.data_ptr(), resid.data_ptr(), ud.numel(),
         dev.stream_handle(ud.device))
    if ud.numel():
        worst = float(resid.max())
        if not worst <= 1e-8:
            k = int(torch.argmax(resid))
            raise NumericalError(
                f"batch quantile failed for {int((resid > 1e-8).sum())} points; worst residual {worst:.3g} "
                f"at u={float(ud[k]):.6g}, nu={nu:g}, lambda={float(ld[k if ld.numel() > 1 else 0]):.6g}")
    return _back(out, u, scalar)


def cir_transition_params(x_prev, kappa, theta, sigma, dt):
    """(nu, lam, scale) of the exact CIR one-step transition (exact_dist.py:542-567)."""
    for name, val in (("kappa", kappa), ("theta", theta), ("sigma", sigma), ("dt", dt)):
        if not (math.isfinite(val) and val > 0.0):
            raise DomainError(f"{name} must be finite and > 0, got {val}")
    x_arr = np.asarray(x_prev, dtype=np.float64)
    if np.any(x_arr < 0.0):
        raise DomainError("x_prev must be >= 0")
    decay = math.exp(-kappa * dt)
    scale = sigma * sigma * (1.0 - decay) / (4.0 * kappa)
    lam = x_arr * (decay / scale)
    nu = 4.0 * kappa * theta / (sigma * sigma)
    if x_arr.ndim == 0:
        lam = float(lam)
    return nu, lam, scale

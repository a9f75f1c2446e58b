"""Exact CIR transition restated in numpy/scipy (TEST INFRASTRUCTURE ONLY).

Restates, for the checker:
  * exact_dist.ncchi2_inv_cdf_batch, per-element-lambda path
    (exact_dist.py:381-434, :451-460) with _vector_newton (:348-378) and the
    Bessel-form density (:416-432) -- scipy.special.chndtr (CDFLIB) and ive
    are the reference's own third-party dependencies (scipy, unpinned
    ``scipy>=1.10`` at pkg/pyproject.toml:10; 1.18.1 in this image);
  * mlmc.simulate_cir_coupled, scheme cir_exact (mlmc.py:253-287), with the
    uniform of step k / path p = PCG32 output k*n_paths + p mapped to
    (w + 0.5) 2^-32.
Pinned by tests/test_oracle.py against the reference's own simulate output
(tests/golden, make_golden.py).
"""

from __future__ import annotations

import math

import numpy as np
from scipy import special as sp

from . import oracle

_LN2 = math.log(2.0)


def _pdf(x, nu, lam):
    order = 0.5 * nu - 1.0
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        dens = 0.5 * np.exp(-0.5 * (np.sqrt(x) - np.sqrt(lam)) ** 2) * (x / lam) ** (0.5 * order) \
            * sp.ive(order, np.sqrt(lam * x))
    small = lam < 1e-10
    if np.any(small):
        a = 0.5 * nu
        with np.errstate(divide="ignore"):
            dens[small] = np.exp((a - 1.0) * np.log(x[small]) - 0.5 * x[small] - a * _LN2 - math.lgamma(a))
    return dens


def ncchi2_inv_cdf_batch(u, nu, lam, x0, tol=1e-9, max_iter=80):
    """Per-element-lambda quantile; returns (x, |chndtr(x) - u|)."""
    u = np.asarray(u, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    hi = lam + nu + 20.0 * np.sqrt(2.0 * (lam + nu)) + 100.0
    tol_f = np.minimum(tol, np.maximum(1e-13, 1e-4 * np.minimum(u, 1.0 - u)))
    guess = np.clip(np.asarray(x0, dtype=np.float64), 1e-8, hi)
    x = np.clip(guess.copy(), 1e-300, hi)
    lo_b = np.zeros_like(x)
    hi_b = hi.copy()
    active = np.arange(x.size)
    for _ in range(max_iter):
        xa = x[active]
        f = sp.chndtr(xa, nu, lam[active]) - u[active]
        ok = np.abs(f) <= tol_f[active]
        if np.all(ok):
            break
        rem = active[~ok]
        f = f[~ok]
        xa = x[rem]
        above = f > 0.0
        hi_b[rem[above]] = xa[above]
        lo_b[rem[~above]] = xa[~above]
        d = _pdf(xa, nu, lam[rem])
        with np.errstate(divide="ignore", invalid="ignore"):
            xn = xa - f / d
        bad = ~np.isfinite(xn) | (xn <= lo_b[rem]) | (xn >= hi_b[rem])
        xn[bad] = 0.5 * (lo_b[rem][bad] + hi_b[rem][bad])
        x[rem] = xn
        active = rem
    resid = np.abs(sp.chndtr(x, nu, lam) - u)
    return x, resid


def cir_exact_paths(*, kappa, theta, sigma, x0, t_end, level, n0, stacks, nu_table, seed, seq, n_paths):
    """(x_exact, x_approx) terminal states per path, mlmc.py:253-287."""
    n_f = n0 << level
    dt = t_end / n_f
    decay = math.exp(-kappa * dt)
    scale = sigma * sigma * (1.0 - decay) / (4.0 * kappa)
    nu = 4.0 * kappa * theta / (sigma * sigma)
    dos = math.exp(-kappa * dt) / scale
    x_e = np.full(n_paths, x0)
    x_a = np.full(n_paths, x0)
    worst = 0.0
    for k in range(n_f):
        w = oracle.pcg32_words(seed, seq, k * n_paths, n_paths)
        u = (w.astype(np.float64) + 0.5) * 2.0**-32
        lam_a = np.maximum(x_a, 0.0) * dos
        x_a = scale * oracle.ncchi2_eval(stacks, nu_table, u, lam_a)
        lam_e = x_e * dos
        warm = oracle.ncchi2_eval(stacks, nu_table, u, lam_e)
        q, resid = ncchi2_inv_cdf_batch(u, nu, lam_e, warm)
        worst = max(worst, float(resid.max()))
        x_e = scale * q
    return x_e, x_a, worst

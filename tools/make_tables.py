"""Generate the shipped approximation tables with the REFERENCE's own fitters.

Tables are offline CPU products that the hot path consumes as-is (SURVEY.md
§2, "Fitting: OUT OF SCOPE").  This script runs only in the build container,
where /root/reference exists; its output ``paper_2012_09715_b200/data/
tables.npz`` is committed, so the GPU box never needs the reference.

Tables written (all float64, reference layouts unless noted):
  constant_q10_l1        fit.fit_constant(10, "l1")                 (1024,)
  dyadic_linear_k15      fit.fit_gaussian_dyadic(1, 15).coeffs      (2, 16)
  dyadic_cubic_k15       fit.fit_gaussian_dyadic(3, 15).coeffs      (4, 16)
  subdyadic_linear_k16_s8  NEW layout (2, 16, 8): octaves j=1..15 of
                         [2^-(j+1), 2^-j) split into 8 equal parts, each an
                         L2 fit by fit.fit_poly_interval (fit.py:227-269);
                         octave 16 = singular remainder (0, 2^-16) with the
                         closed-form fit (fit.py:66-73, :292-296), replicated
                         over its 8 slots.
  ncchi2_nu{tag}_k{n}_stacks  fit.fit_ncchi2(nu, n_knots=n).eval_stacks
                         (2, n, 2, 16) plus the nu value.

Usage:  python tools/make_tables.py [--out PATH] [--skip-ncchi2]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"


def _import_reference():
    os.environ.setdefault("APPROXRV_BACKEND", "python")  # bitwise-identical numpy kernels
    sys.path.insert(0, REF_SRC)
    import approxrv  # noqa: F401
    from approxrv import fit

    return fit


def subdyadic_linear(fit, K: int = 16, sub_bits: int = 3, degree: int = 1) -> np.ndarray:
    oracle = fit.GaussianQuantileOracle()
    nsub = 1 << sub_bits
    coeffs = np.zeros((degree + 1, K, nsub))
    for j in range(1, K):
        a = 2.0 ** -(j + 1)
        h = a / nsub
        for s in range(nsub):
            lo = a + s * h
            hi = a + (s + 1) * h
            coeffs[:, j - 1, s] = fit.fit_poly_interval(lo, hi, degree, oracle)
    b_last = 2.0 ** -K
    if degree == 1:
        alpha, beta = oracle.singular_linear_fit(b_last)
        coeffs[0, K - 1, :] = alpha
        coeffs[1, K - 1, :] = beta
    else:
        coeffs[:, K - 1, :] = fit.fit_poly_interval(0.0, b_last, degree, oracle)[:, None]
    return coeffs


def main() -> None:
    ap = argparse.ArgumentParser()
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ap.add_argument("--out", default=os.path.join(here, "paper_2012_09715_b200", "data", "tables.npz"))
    ap.add_argument("--skip-ncchi2", action="store_true")
    args = ap.parse_args()
    fit = _import_reference()
    t = {}
    t0 = time.time()
    t["constant_q10_l1"] = fit.fit_constant(10, "l1").values
    t["dyadic_linear_k15"] = fit.fit_gaussian_dyadic(1, 15).coeffs
    t["dyadic_cubic_k15"] = fit.fit_gaussian_dyadic(3, 15).coeffs
    t["subdyadic_linear_k16_s8"] = subdyadic_linear(fit, 16, 3, 1)
    print(f"gaussian tables: {time.time() - t0:.1f}s", flush=True)
    if not args.skip_ncchi2:
        # CIR defaults of BASELINE.json config 5 / cli.py:273 (nu is 1.9999999999999996).
        kappa, theta, sigma = 0.5, 0.04, 0.2
        nu = 4.0 * kappa * theta / sigma**2
        for n_knots in (16, 64):
            t1 = time.time()
            tab = fit.fit_ncchi2(nu, n_knots=n_knots, m=1, n_intervals=15)
            t[f"ncchi2_cir_k{n_knots}_stacks"] = tab.eval_stacks
            t[f"ncchi2_cir_k{n_knots}_nu"] = np.float64(tab.nu)
            print(f"ncchi2 nu={nu!r} knots={n_knots}: {time.time() - t1:.1f}s", flush=True)
        t1 = time.time()
        tab = fit.fit_ncchi2(1.0, n_knots=16, m=1, n_intervals=15)
        t["ncchi2_nu1_k16_stacks"] = tab.eval_stacks
        t["ncchi2_nu1_k16_nu"] = np.float64(1.0)
        print(f"ncchi2 nu=1 knots=16: {time.time() - t1:.1f}s", flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    np.savez_compressed(args.out, **t)
    print("wrote", args.out, {k: np.shape(v) for k, v in t.items()})


if __name__ == "__main__":
    main()

"""Device throughput of the drop-in plugin kernels (_kernels.pyx replacements).

Each kernel reads its input once and writes its output once; the roofline is
the measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs).

    python tools/bench_dropin.py [--n 268435456] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200 import _kernels as k  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    n = args.n
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    u64 = arv.PhiloxStream(1, 2).uniforms(n)
    u32 = u64.float()
    o64 = torch.empty_like(u64)
    o32 = torch.empty_like(u32)
    lin = arv.load_table("dyadic_linear_k15")
    cub = arv.load_table("dyadic_cubic_k15")
    const = arv.load_table("constant_q10_l1")
    sub = arv.load_table("subdyadic_linear_k16_s8")
    nc = arv.load_table("ncchi2_cir_k64_stacks")
    lam1 = torch.full((1,), 7.5, dtype=torch.float64, device="cuda")
    lamn = u64 * 300.0
    cases = {
        "constant_eval f64": (lambda: k.constant_eval(const.values, u64, o64), 16),
        "dyadic_eval f64 linear": (lambda: k.dyadic_eval(lin.coeffs, u64, o64), 16),
        "dyadic_eval f64 cubic": (lambda: k.dyadic_eval(cub.coeffs, u64, o64), 16),
        "dyadic_eval32 linear": (lambda: k.dyadic_eval32(lin.coeffs32, u32, o32), 8),
        "subdyadic_eval32 16x8": (lambda: k.subdyadic_eval32(sub.coeffs32, 3, u32, o32), 8),
        "dyadic_index f64": (lambda: k.dyadic_index(u64, 15), 16),
        "ncchi2_eval shared lam": (lambda: k.ncchi2_eval(nc.eval_stacks, nc.nu, u64, lam1, o64), 16),
        "ncchi2_eval per-element lam": (lambda: k.ncchi2_eval(nc.eval_stacks, nc.nu, u64, lamn, o64), 24),
        "gaussian_inv_cdf f64": (lambda: k.gaussian_inv_cdf(u64, o64), 16),
        "gaussian_inv_cdf32": (lambda: k.gaussian_inv_cdf32(u32, o32), 8),
        "torch copy f64 (reference)": (lambda: o64.copy_(u64), 16),
    }
    for name, (fn, bps) in cases.items():
        s = timed(fn, args.reps)
        gbs = n * bps / s / 1e9
        print(json.dumps({"kernel": name, "n": n, "ms": s * 1e3, "samples_per_s": n / s, "bytes_per_sample": bps,
                          "gbs": gbs, "frac_copy_peak": gbs / peak}), flush=True)


if __name__ == "__main__":
    main()

"""Throughput of the SURVEY §8(f) rows built after the hot path, on one B200:

* Philox-4x64-10 replay of the reference's UniformStream (`PhiloxStream`):
  raw words, f64 uniforms, fused K15 dyadic f64 and AS241 f64 samples, 2^28
  outputs of 8 B each -> samples/s and fraction of the copy peak;
* device ncchi2 quantile (`exact_dist.ncchi2_inv_cdf_batch`, per-element lambda)
  and the Table-5 style `metrics.rmse_ncchi2` grid;
* the reference's CPU `UniformStream.uniforms` rate for comparison is in
  SURVEY §8(a) (39 ns/sample, one thread).

    python tools/bench_next_rows.py > profiles/r01_next_rows.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200 import exact_dist, metrics  # noqa: E402


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
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    n = 1 << 28
    out64 = torch.empty(n, dtype=torch.float64, device="cuda")
    lin = arv.load_table("dyadic_linear_k15")
    ph = arv.PhiloxStream(42, 7)
    cases = {
        "philox raw_words": (lambda: ph.raw_words(n), 8),
        "philox uniforms f64": (lambda: ph.uniforms(n, out=out64), 8),
        "philox -> dyadic K15 f64": (lambda: ph.sample(lin, n, out=out64), 8),
        "philox -> AS241 f64": (lambda: ph.sample("exact", n, out=out64), 8),
    }
    for name, (fn, bps) in cases.items():
        s = timed(fn, 10)
        print(json.dumps({"case": name, "n": n, "ms": s * 1e3, "samples_per_s": n / s,
                          "gbs": n * bps / s / 1e9, "frac_copy_peak": n * bps / s / 1e9 / peak}), flush=True)
    del out64
    # device exact ncchi2 quantile, per-element lambda (the CIR transition law)
    m = 1 << 22
    g = torch.Generator(device="cuda").manual_seed(3)
    u = torch.rand(m, dtype=torch.float64, device="cuda", generator=g).clamp_(1e-12, 1 - 1e-12)
    lam = torch.rand(m, dtype=torch.float64, device="cuda", generator=g) * 400.0
    nu = 4 * 0.5 * 0.04 / 0.2 ** 2
    s = timed(lambda: exact_dist.ncchi2_inv_cdf_batch(u, nu, lam), 3)
    print(json.dumps({"case": "ncchi2_inv_cdf_batch per-element lambda in [0,400), no warm start", "n": m,
                      "ms": s * 1e3, "quantiles_per_s": m / s}), flush=True)
    tab = arv.load_table("ncchi2_cir_k64_stacks")
    grid = [0.5, 1.0, 2.0, 5.0, 10.0, 20.0, 50.0, 100.0, 200.0]
    s = timed(lambda: metrics.rmse_ncchi2(tab, grid, 10 ** 5), 2)
    print(json.dumps({"case": "rmse_ncchi2 (64-knot CIR table, 9 lambdas x 1e5 lattice points)",
                      "ms": s * 1e3, "cells": len(grid)}), flush=True)


if __name__ == "__main__":
    main()

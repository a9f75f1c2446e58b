"""BASELINE.json config 3: exact vs approximate throughput sweep on one B200.

Fused PCG32 generation for N = 2^20 ... 2^32 samples of
  constant q10 (config 1 table), dyadic K15 linear (reference layout),
  16x8 sub-interval linear (config 2), AS241 in f32, AS241 in f64,
reporting samples/s (CUDA events, best of R after warm-up) and, for the
HBM-bound generators, the fraction of the measured copy peak.

    python tools/sweep_config3.py [--max-log2 32] [--reps 5] > profiles/r01_config3_sweep.jsonl
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2012_09715_b200 as arv  # noqa: E402


def best_ms(fn, reps):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=20)
    ap.add_argument("--max-log2", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    hbm = peaks.get("hbm_gbs", 6650.0)
    nmax = 1 << args.max_log2
    out32 = torch.empty(nmax, dtype=torch.float32, device="cuda")
    out64 = torch.empty(nmax, dtype=torch.float64, device="cuda")
    tabs = {
        "constant_q10": arv.load_table("constant_q10_l1"),
        "dyadic_k15_linear": arv.load_table("dyadic_linear_k15"),
        "subdyadic_16x8_linear": arv.load_table("subdyadic_linear_k16_s8"),
    }
    for lg in range(args.min_log2, args.max_log2 + 1):
        n = 1 << lg
        row = {"log2_n": lg, "n": n}
        for name, t in tabs.items():
            ms = best_ms(lambda: arv.Pcg32Stream(42, 0).sample(t, n, out=out32[:n]), args.reps)
            row[name] = {"samples_per_s": n / ms * 1e3, "ms": ms, "gbs": 4 * n / ms / 1e6,
                         "frac_copy_peak": 4 * n / ms / 1e6 / hbm}
        ms = best_ms(lambda: arv.Pcg32Stream(42, 0).sample("exact", n, out=out32[:n]), args.reps)
        row["as241_f32"] = {"samples_per_s": n / ms * 1e3, "ms": ms}
        ms = best_ms(lambda: arv.Pcg32Stream(42, 0).sample_exact64(n, out=out64[:n]), args.reps)
        row["as241_f64"] = {"samples_per_s": n / ms * 1e3, "ms": ms}
        print(json.dumps(row), flush=True)
    print(json.dumps({"accuracy": accuracy(tabs)}), flush=True)


def accuracy(tabs, n=1 << 24):
    """Errors against AS241 in f64 on the same f32 lattice uniforms (the fused
    generators' inputs): the f32 AS241 evaluation (max relative error and f32
    ulps) and each table approximation (RMSE, max |error|)."""
    from paper_2012_09715_b200 import _kernels

    u = arv.Pcg32Stream(42, 0).uniforms(n)                      # f32 lattice
    ref = torch.empty(n, dtype=torch.float64, device="cuda")
    _kernels.gaussian_inv_cdf(u.double(), ref)                  # AS241 f64 of the same u
    z32 = arv.Pcg32Stream(42, 0).sample("exact", n)             # AS241 in f32 (fused)
    d = z32.double() - ref
    rel = (d.abs() / ref.abs().clamp_min(1e-300)).max().item()
    ulp = (d.abs() / (torch.nextafter(z32.abs(), torch.tensor(float("inf"), device="cuda")) - z32.abs()).double()).max().item()
    res = {"samples": n, "as241_f32_vs_f64": {"max_rel": rel, "max_abs": d.abs().max().item(), "max_f32_ulp": ulp}}
    for name, t in tabs.items():
        e = arv.Pcg32Stream(42, 0).sample(t, n).double() - ref
        res[name] = {"rmse": torch.sqrt((e * e).mean()).item(), "max_abs": e.abs().max().item()}
    return res


if __name__ == "__main__":
    main()

"""Launch each hot kernel a few times (for ncu captures; prints CUDA-event times).

    python tools/prof_kernels.py [--which sub,const,store,gauss64,gbm,cir] [--reps 3]
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200 import _native  # noqa: E402
from paper_2012_09715_b200.mlmc import run_level  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def sweep(args):
    n = args.n
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    t = arv.load_table("subdyadic_linear_k16_s8")
    c = arv.load_table("constant_q10_l1")
    for group in (4, 8):
        for ctas in (2, 4, 6, 8):
            _native.call("arv_set_tuning", 1, group)
            _native.call("arv_set_tuning", 2, ctas)
            r = {
                "sub": timed(lambda: arv.Pcg32Stream(42, 0).sample(t, n, out=out), args.reps),
                "const": timed(lambda: arv.Pcg32Stream(42, 0).sample(c, n, out=out), args.reps),
                "words": timed(lambda: arv.Pcg32Stream(42, 0).words(n, out=out.view(torch.uint32)), args.reps),
                "store": timed(lambda: _native.call("arv_store_probe_ex", out.data_ptr(), n, group, s), args.reps),
            }
            print(f"group={group} ctas={ctas} " + " ".join(f"{k}={v:.4f}ms({n * 4 / v / 1e6:.0f}GB/s)"
                                                          for k, v in r.items()), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="sub,const,store,gauss64,gbm,cir")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--group", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--cirseg", type=int, default=-1, help="CIR exact steps per segment (0: one kernel)")
    args = ap.parse_args()
    if args.cirseg >= 0:
        _native.call("arv_set_tuning", 3, args.cirseg)
    if args.group:
        _native.call("arv_set_tuning", 1, args.group)
    if args.ctas:
        _native.call("arv_set_tuning", 2, args.ctas)
    if args.sweep:
        return sweep(args)
    which = args.which.split(",")
    n = args.n
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    if "sub" in which:
        t = arv.load_table("subdyadic_linear_k16_s8")
        res["sub"] = timed(lambda: arv.Pcg32Stream(42, 0).sample(t, n, out=out), args.reps)
    if "k15" in which:
        t = arv.load_table("dyadic_linear_k15")
        res["k15"] = timed(lambda: arv.Pcg32Stream(42, 0).sample(t, n, out=out), args.reps)
    if "const" in which:
        t = arv.load_table("constant_q10_l1")
        res["const"] = timed(lambda: arv.Pcg32Stream(42, 0).sample(t, n, out=out), args.reps)
    if "store" in which:
        for m in (4, 5, 8):
            res[f"store_m{m}"] = timed(lambda: _native.call("arv_store_probe_ex", out.data_ptr(), n, m, s), args.reps)
    if "words" in which:
        o = out.view(torch.uint32)
        res["words"] = timed(lambda: arv.Pcg32Stream(42, 0).words(n, out=o), args.reps)
    if "gauss32" in which:
        res["gauss32"] = timed(lambda: arv.Pcg32Stream(42, 0).sample("exact", n, out=out), args.reps)
    if "gauss64" in which:
        o64 = torch.empty(n // 2, dtype=torch.float64, device="cuda")
        res["gauss64"] = timed(lambda: arv.Pcg32Stream(42, 0).sample_exact64(n // 2, out=o64), args.reps)
    if "gbm" in which:
        lin = arv.load_table("dyadic_linear_k15")
        sp = arv.LevelSpec(level=8, scheme="euler_maruyama", process=arv.GbmParams(0.05, 0.2, 1.0, 1.0),
                           rv_source=lin, kind="four_way", n0=1)
        res["gbm_l8"] = timed(lambda: run_level(sp, arv.level_stream(42, 8), 1 << 22), args.reps)
    if "gbml01" in which:  # levels 0 and 1 of config 4 (per-level fixed cost)
        lin = arv.load_table("dyadic_linear_k15")
        for lv in (0, 1):
            sp = arv.LevelSpec(level=lv, scheme="euler_maruyama", process=arv.GbmParams(0.05, 0.2, 1.0, 1.0),
                               rv_source=lin, kind="four_way", n0=1)
            res[f"gbm_l{lv}"] = timed(lambda: run_level(sp, arv.level_stream(42, lv), 1 << 22), args.reps)
    if "gbmall" in which:  # config 4: levels 0..8 x 2^22 paths, level kernel + merge each
        lin = arv.load_table("dyadic_linear_k15")
        sps = [arv.LevelSpec(level=lv, scheme="euler_maruyama", process=arv.GbmParams(0.05, 0.2, 1.0, 1.0),
                             rv_source=lin, kind="four_way", n0=1) for lv in range(9)]
        res["gbm_all"] = timed(lambda: [run_level(sp, arv.level_stream(42, sp.level), 1 << 22) for sp in sps],
                               args.reps)
    if "cir" in which:
        tab = arv.load_table("ncchi2_cir_k64_stacks")
        sp = arv.LevelSpec(level=6, scheme="cir_exact", process=arv.CirParams(0.5, 0.04, 0.2, 0.04, 1.0),
                           rv_source=tab, kind="four_way", n0=1)
        res["cir_l6"] = timed(lambda: run_level(sp, arv.level_stream(42, 6), 1 << 20), args.reps)
    if "cirall" in which:  # config 5: every level, 2^20 paths
        tab = arv.load_table("ncchi2_cir_k64_stacks")
        for lv in range(7):
            sp = arv.LevelSpec(level=lv, scheme="cir_exact", process=arv.CirParams(0.5, 0.04, 0.2, 0.04, 1.0),
                               rv_source=tab, kind="four_way", n0=1)
            res[f"cir_l{lv}"] = timed(lambda: run_level(sp, arv.level_stream(42, lv), 1 << 20), args.reps)
    for k, v in res.items():
        print(f"{k}: {v:.4f} ms")


if __name__ == "__main__":
    main()

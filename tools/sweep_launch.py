"""Launch-shape sweep of the fused generators at one size, each launch timed
alone after an L2 flush (512 MiB store sweep) or back to back.

    python tools/sweep_launch.py --n 16777216 --flush --ctas 4,6,8,12,16,24 --group 4,8
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200 import _native  # noqa: E402


def per_launch(fn, reps, scratch):
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if scratch is None:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps * 1e-3
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        _native.call("arv_store_probe", scratch.data_ptr(), scratch.numel(), s)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--ctas", default="0,4,6,8,12,16")  # 0 = auto
    ap.add_argument("--group", default="4,8")
    args = ap.parse_args()
    n = args.n
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    scratch = torch.empty(128 << 20, dtype=torch.float32, device="cuda") if args.flush else None
    sub = arv.load_table("subdyadic_linear_k16_s8")
    const = arv.load_table("constant_q10_l1")
    for group in [int(x) for x in args.group.split(",")]:
        for ctas in [int(x) for x in args.ctas.split(",")]:
            _native.call("arv_set_tuning", 1, group)
            _native.call("arv_set_tuning", 2, ctas)
            r = {"n": n, "flush": args.flush, "group": group, "ctas": ctas}
            for name, t in (("sub", sub), ("const", const)):
                sec = per_launch(lambda: arv.Pcg32Stream(42, 0).sample(t, n, out=out), args.reps, scratch)
                r[name + "_us"] = sec * 1e6
                r[name + "_per_s"] = n / sec
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()

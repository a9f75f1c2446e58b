"""Per-level kernel time of the config-4 (GBM EM, 2^22 paths) and config-5 (CIR
exact, 2^20 paths) pilots, against the path-step-proportional ideal taken from the
longest level: the remainder is per-level fixed cost (launch, path setup, merge)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200.mlmc import run_level  # noqa: E402


def per_level(specs, n, reps=5):
    out = []
    for sp in specs:
        run_level(sp, arv.level_stream(42, sp.level), n)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            run_level(sp, arv.level_stream(42, sp.level), n)
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b) / reps)
    return out


def main():
    lin = arv.load_table("dyadic_linear_k15")
    cir = arv.load_table("ncchi2_cir_k64_stacks")
    for name, specs, n in (
        ("gbm", [arv.LevelSpec(level=l, scheme="euler_maruyama", process=arv.GbmParams(0.05, 0.2, 1.0, 1.0),
                               rv_source=lin, kind="four_way", n0=1) for l in range(9)], 1 << 22),
        ("cir", [arv.LevelSpec(level=l, scheme="cir_exact", process=arv.CirParams(0.5, 0.04, 0.2, 0.04, 1.0),
                               rv_source=cir, kind="four_way", n0=1) for l in range(7)], 1 << 20),
    ):
        t = per_level(specs, n)
        top = len(t) - 1
        unit = t[top] / (1 << top)
        for l, ms in enumerate(t):
            print(f"{name} l{l}: {ms:.4f} ms  (ideal {unit * (1 << l):.4f}, fixed {ms - unit * (1 << l):+.4f})")
        print(f"{name} total {sum(t):.3f} ms, ideal {unit * ((1 << len(t)) - 1):.3f} ms")


if __name__ == "__main__":
    main()

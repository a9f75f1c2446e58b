"""Headline generator launch-shape / build-variant tuning on the GPU box.

Burst: mean of 20 back-to-back 2^28 launches (after warm-up) for CTAs-per-SM
settings (0 = the library's auto policy); sustained: the bench's 2 s leg
(launches in t = 1..2 s) at the auto setting, with NVML clocks.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200 import _native  # noqa: E402


def main():
    n = 1 << 28
    t = arv.load_table("subdyadic_linear_k16_s8")
    out = torch.empty(n, dtype=torch.float32, device="cuda")

    def step():
        arv.Pcg32Stream(42, 0).sample(t, n, out=out)

    lib = os.path.basename(os.environ.get("ARV_LIB_PATH", "in-tree"))
    res = []
    for ctas in (0, 4, 6, 8, 10, 12):
        _native.call("arv_set_tuning", 2, ctas)
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            step()
        b.record()
        b.synchronize()
        res.append(f"ctas={ctas}:{a.elapsed_time(b) / 20 * 1e3:.1f}us")
    _native.call("arv_set_tuning", 2, 0)
    sus, clk = bench.sustained_per_launch(step, torch.device("cuda", 0), seconds=2.0)
    print(f"{lib}: burst " + " ".join(res) + f" | sustained {sus * 1e6:.1f}us {n / sus:.3e}/s "
          f"sm {clk['sm_mhz']} {clk['reasons']}", flush=True)


if __name__ == "__main__":
    main()

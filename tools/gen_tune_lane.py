"""Headline generator: signed-table kernel vs lane-table kernel (ARV_TUNE_LANE_MIN_N).

    python tools/gen_tune_lane.py <lane_min_n_log2: -1 = signed kernel, 24 / 26 = lane kernel> [ctas_per_sm]

One variant per process, so that the burst figure (200 back-to-back 2^28
launches from an idle GPU, as bench.py) is not taken at the power cap the
previous variant's sustained leg (2 s) left behind."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200 import _native  # noqa: E402


def main():
    lm = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    n = 1 << 28
    t = arv.load_table("subdyadic_linear_k16_s8")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    _native.call("arv_set_tuning", 5, lm)
    _native.call("arv_set_tuning", 2, ctas)

    def step():
        arv.Pcg32Stream(42, 0).sample(t, n, out=out)

    res = []
    for rep in range(3):
        time.sleep(1.0)  # idle: clocks and power back to the burst state
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(200):
            step()
        b.record()
        b.synchronize()
        res.append(f"{a.elapsed_time(b) / 200 * 1e3:.1f}")
    sus, clk = bench.sustained_per_launch(step, torch.device("cuda", 0), seconds=2.0)
    print(f"lane_min_n={lm} ctas={ctas}: burst(200 launches) {'/'.join(res)} us | sustained {sus * 1e6:.1f}us "
          f"{n / sus:.3e}/s sm {clk['sm_mhz']} {clk['reasons']}", flush=True)


if __name__ == "__main__":
    main()

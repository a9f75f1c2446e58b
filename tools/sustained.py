"""Sustained vs burst throughput of the headline generator: back-to-back
launches for --seconds, timed in windows of --window launches with CUDA
events, with NVML SM clock / power / throttle reasons sampled per window.

    python tools/sustained.py [--n 268435456] [--seconds 5] [--window 50] [--kernel sub|const|words|store]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--seconds", type=float, default=5.0)
    ap.add_argument("--window", type=int, default=50)
    ap.add_argument("--kernel", default="sub")
    args = ap.parse_args()
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    n = args.n
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    if args.kernel == "store":
        fn = lambda: _native.call("arv_store_probe", out.data_ptr(), n, s)  # noqa: E731
    elif args.kernel == "words":
        fn = lambda: arv.Pcg32Stream(42, 0).words(n, out=out.view(torch.uint32))  # noqa: E731
    else:
        t = arv.load_table("subdyadic_linear_k16_s8" if args.kernel == "sub" else "constant_q10_l1")
        fn = lambda: arv.Pcg32Stream(42, 0).sample(t, n, out=out)  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    total = 0.0
    w = 0
    while total < args.seconds:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.window):
            fn()
        b.record()
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mem = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
        tr = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        temp = pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)
        b.synchronize()
        dt = a.elapsed_time(b) * 1e-3
        total += dt
        print(json.dumps({"window": w, "t_end_s": total, "us_per_launch": dt / args.window * 1e6,
                          "gbs": n * 4 * args.window / dt / 1e9, "sm_mhz": sm, "mem_mhz": mem, "power_w": pw,
                          "temp_c": temp, "throttle_mask": hex(tr)}), flush=True)
        w += 1


if __name__ == "__main__":
    main()

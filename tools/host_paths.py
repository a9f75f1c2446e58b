"""Host-side costs of the public APIs on the GPU box.

* PCIe ceilings: pinned H2D / D2H / bidirectional copy bandwidth (torch).
* the numpy plugin pipeline (_kernels.dyadic_eval32 on 2^28 f32 host arrays)
  for ARV_HOST_THREADS-like pool sizes (set per process via env; this tool
  re-executes itself per setting).
* estimate_level_suites host overhead: wall clock vs device time, cProfile top.
"""
import cProfile
import io
import os
import pstats
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def pcie():
    n = 1 << 28
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    d2 = torch.empty(n, dtype=torch.float32, device="cuda")
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        print(f"pcie {name}: {5 * n * 4 / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    print(f"pcie bidirectional: {5 * n * 4 / (time.perf_counter() - t) / 1e9:.1f} GB/s each way", flush=True)
    a = np.ones(n, np.float32)
    b = np.empty(n, np.float32)
    b.fill(0)
    t = time.perf_counter()
    np.copyto(b, a)
    print(f"host memcpy 1 thread: {n * 4 / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)


def plugin():
    import paper_2012_09715_b200 as arv
    from paper_2012_09715_b200 import _kernels

    n = 1 << 28
    lin = arv.load_table("dyadic_linear_k15")
    u = arv.Pcg32Stream(42, 0).uniforms(n).cpu().numpy()
    out = np.empty(n, np.float32)
    out.fill(0)
    _kernels.dyadic_eval32(lin.coeffs32, u[:1 << 20], out[:1 << 20])
    t = time.perf_counter()
    for _ in range(3):
        _kernels.dyadic_eval32(lin.coeffs32, u, out)
    dt = (time.perf_counter() - t) / 3
    print(f"plugin threads={os.environ.get('ARV_HOST_THREADS', 'default')}: {dt * 1e3:.1f} ms = {n / dt:.3e} "
          f"samples/s ({2 * n * 4 / dt / 1e9:.1f} GB/s host<->device total)", flush=True)


def suites():
    import paper_2012_09715_b200 as arv

    lin = arv.load_table("dyadic_linear_k15")
    specs = [arv.LevelSpec(level=l, scheme="euler_maruyama", process=arv.GbmParams(0.05, 0.2, 1.0, 1.0),
                           rv_source=lin, kind="four_way", n0=1) for l in range(9)]
    streams = [arv.level_stream(42, sp.level) for sp in specs]
    arv.estimate_level_suites(specs, streams, 1 << 22)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    res = arv.estimate_level_suites(specs, streams, 1 << 22)
    e1.record()
    e1.synchronize()
    wall = time.perf_counter() - t
    dev = sum(r["four_way"].cost_per_path_seconds * r["four_way"].n_paths for r in res)
    print(f"suites: wall {wall * 1e3:.2f} ms, events {e0.elapsed_time(e1):.2f} ms, sum of level intervals "
          f"{dev * 1e3:.2f} ms", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        arv.estimate_level_suites(specs, streams, 1 << 22)
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14)
    print(s.getvalue()[-3500:])


def graph():
    """Per-call cost of small fused-generator requests: eager calls (Python +
    ctypes + launch each) vs the same calls replayed from one CUDA graph."""
    import paper_2012_09715_b200 as arv

    sub = arv.load_table("subdyadic_linear_k16_s8")
    for lg in (16, 20, 24):
        n, k = 1 << lg, 64
        out = torch.empty((k, n), dtype=torch.float32, device="cuda")
        s = arv.Pcg32Stream(42, 0)
        for i in range(k):
            s.sample(sub, n, out=out[i])
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            for i in range(k):
                s.sample(sub, n, out=out[i])
        torch.cuda.synchronize()
        eager = (time.perf_counter() - t) / (5 * k)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(k):
                s.sample(sub, n, out=out[i])
        g.replay()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        replay = (time.perf_counter() - t) / (5 * k)
        print(f"2^{lg} samples per call: eager {eager * 1e6:.2f} us/call, graph replay {replay * 1e6:.2f} us/call "
              f"({n / replay:.3e} samples/s)", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "all":
        pcie()
        for th in ("8", "16"):
            subprocess.run([sys.executable, __file__, "plugin"], env=dict(os.environ, ARV_HOST_THREADS=th))
        suites()
        graph()
    else:
        globals()[what]()

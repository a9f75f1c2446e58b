import sys, torch
sys.path.insert(0, '.')
import paper_2012_09715_b200 as arv
from paper_2012_09715_b200 import _native
t = arv.load_table("subdyadic_linear_k16_s8")
for lg in range(19, 27):
    n = 1 << lg
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    res = []
    for lm in (-1, 0):
        _native.call("arv_set_tuning", 5, lm)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                arv.Pcg32Stream(42, 0).sample(t, n, out=out)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for i in range(16):
                    arv.Pcg32Stream(42, 0, counter=i * n).sample(t, n, out=out)
            g.replay(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                g.replay()
            b.record(); b.synchronize()
            res.append(a.elapsed_time(b) / 160 * 1e3)
    print(f"2^{lg}: signed {res[0]:.2f} us  lane {res[1]:.2f} us", flush=True)
_native.call("arv_set_tuning", 5, 24)

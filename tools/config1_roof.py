"""Config 1 (2^24 f32 samples) against the store-only roof at the same size,
each launch timed alone after a 512 MiB L2 flush (as bench.py --workload
config1) and back to back; plus an empty launch for the fixed cost.

    python tools/config1_roof.py
"""
import sys, torch
sys.path.insert(0, '.')
import paper_2012_09715_b200 as arv
from paper_2012_09715_b200 import _native
sys.path.insert(0, 'tools')
from sweep_launch import per_launch
n = 1 << 24
out = torch.empty(n, dtype=torch.float32, device="cuda")
scratch = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
c = arv.load_table("constant_q10_l1")
for name, fn in (("store_probe", lambda: _native.call("arv_store_probe", out.data_ptr(), n, s)),
                 ("const", lambda: arv.Pcg32Stream(42, 0).sample(c, n, out=out)),
                 ("empty_launch(n=8)", lambda: _native.call("arv_store_probe", out.data_ptr(), 8, s))):
    for flush in (scratch, None):
        print(name, "flush" if flush is not None else "noflush", "%.2f us" % (per_launch(fn, 100, flush) * 1e6))

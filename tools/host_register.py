"""Cost of cudaHostRegister / Unregister on numpy buffers (GPU box), and the
pinned-in-place DMA rate from / to them."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

cr = torch.cuda.cudart()
for mib in (64, 256, 1024):
    a = np.ones(mib << 18, np.float32)
    t = time.perf_counter()
    rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t_reg = time.perf_counter() - t
    d = torch.empty(a.size, dtype=torch.float32, device="cuda")
    ta = torch.from_numpy(a)
    d.copy_(ta, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        d.copy_(ta, non_blocking=True)
    torch.cuda.synchronize()
    h2d = 3 * a.nbytes / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    rc2 = cr.cudaHostUnregister(a.ctypes.data)
    t_unreg = time.perf_counter() - t
    print(f"{mib} MiB: register {t_reg * 1e3:.2f} ms (rc {rc}), H2D from registered {h2d:.1f} GB/s, "
          f"unregister {t_unreg * 1e3:.2f} ms (rc {rc2})", flush=True)

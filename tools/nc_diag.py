"""CDF evaluations per exact CIR transition, per level of config 5 (needs the
diagnostic build: _build.build(defines=['ARV_NC_COUNT=1'], out=LIB), run with
ARV_LIB_PATH=LIB)."""

import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200 import _native  # noqa: E402
from paper_2012_09715_b200.mlmc import run_level  # noqa: E402

lib = _native.lib
cnt = (ctypes.c_ulonglong * 18)()
tab = arv.load_table("ncchi2_cir_k64_stacks")
lib.arv_nc_counters(cnt)
for lv in range(7):
    sp = arv.LevelSpec(level=lv, scheme="cir_exact", process=arv.CirParams(0.5, 0.04, 0.2, 0.04, 1.0),
                       rv_source=tab, kind="four_way", n0=1)
    run_level(sp, arv.level_stream(42, lv), 1 << 18)
    torch.cuda.synchronize()
    lib.arv_nc_counters(cnt)
    solves = max(cnt[1], 1)
    lanes = " ".join(f"{k}:{cnt[2 + k] / solves:.4f}" for k in range(1, 8) if cnt[2 + k])
    warps = sum(cnt[10 + k] for k in range(8)) or 1
    wmax = " ".join(f"{k}:{cnt[10 + k] / warps:.4f}" for k in range(1, 8) if cnt[10 + k])
    print(f"level {lv}: {cnt[1]} solves, {cnt[0] / solves:.3f} CDF evaluations per solve; "
          f"per solve {{{lanes}}}; warp max {{{wmax}}}")

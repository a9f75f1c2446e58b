"""Worker for tests/test_gpu_dist.py (launched by torch.distributed.run).

Every rank runs the distributed MLMC pilot (paths sharded over ranks, two
all-reduces of the per-kind triples) and the single-process pilot over all
paths, and checks they agree.  Uses gloo so ranks may share one GPU without
any GPU kernel waiting on another rank.
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out_dir = sys.argv[1]
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    import paper_2012_09715_b200 as arv
    from paper_2012_09715_b200.mlmc import NSLOT, run_level

    res = {}
    cases = [
        ("gbm", arv.LevelSpec(level=4, scheme="euler_maruyama", process=arv.GbmParams(0.05, 0.2, 1.0, 1.0),
                              rv_source=arv.load_table("dyadic_linear_k15"), kind="four_way", n0=1)),
        ("cir", arv.LevelSpec(level=2, scheme="cir_exact", process=arv.CirParams(0.5, 0.04, 0.2, 0.04, 1.0),
                              rv_source=arv.load_table("ncchi2_cir_k64_stacks"), kind="four_way", n0=1)),
    ]
    n = 30011
    for name, spec in cases:
        suite = arv.estimate_level_suite(spec, arv.level_stream(42, spec.level), n)  # sharded (dist detected)
        full, _, _ = run_level(spec, arv.level_stream(42, spec.level), n)             # this rank, all paths
        full = full.cpu().numpy()
        keys = list(suite)
        slot = {"two_way_exact": 0, "two_way_approx": 1, "four_way": 2, "plain_exact": 3, "plain_approx": 4,
                "correction": 2}
        for k in keys:
            s = suite[k]
            f = full[slot[k]]
            res[f"{name}/{k}"] = [s.n_paths, s.mean, s.variance, f[0], f[1], f[2] / (f[0] - 1)]
        assert full.shape == (NSLOT, 3)
    # the batched pilot (all levels, one all-reduce pair) equals the per-level calls
    specs = [spec for _, spec in cases]
    suites = arv.estimate_level_suites(specs, [arv.level_stream(42, sp.level) for sp in specs], n)
    for (name, spec), got in zip(cases, suites):
        want = arv.estimate_level_suite(spec, arv.level_stream(42, spec.level), n)
        for k in want:
            assert (got[k].n_paths, got[k].mean, got[k].variance) == \
                (want[k].n_paths, want[k].mean, want[k].variance), (name, k)
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
        json.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()
    _ = np


if __name__ == "__main__":
    main()

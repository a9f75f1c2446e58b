"""Small invocation of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) on the GPU box:

    compute-sanitizer --tool racecheck python tools/sanitize.py

Covers the fused generators (v8 / v4 / scalar store paths, signed-table, lane-table and
general evaluators, PDL launch), the lattice hook, the Gaussian level kernels
(v2 with the warp-wide AS241 tail list; the Philox kernel), the atomic-ticket
chunk finalize (more than 2048 CTA partials), the CIR exact level in its
one-kernel CTA-sorted form and its segmented form (bucket scan + scatter),
the standalone ncchi2 quantile / CDF, AS241, the drop-in element-wise
kernels and the host-buffer pipeline.  Sizes are small: the tools slow
kernels down by 10-100x.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_09715_b200 as arv  # noqa: E402
from paper_2012_09715_b200 import _kernels, _native  # noqa: E402
from paper_2012_09715_b200.mlmc import run_level  # noqa: E402


def main():
    big = "--big" in sys.argv
    n = (1 << 20) + 3 if big else (1 << 16) + 3
    sub = arv.load_table("subdyadic_linear_k16_s8")
    const = arv.load_table("constant_q10_l1")
    lin = arv.load_table("dyadic_linear_k15")
    cub = arv.load_table("dyadic_cubic_k15")
    buf = torch.empty(n + 8, dtype=torch.float32, device="cuda")
    for t in (sub, const, lin, cub):
        arv.Pcg32Stream(42, 0).sample(t, n, out=buf[:n])           # v8
        arv.Pcg32Stream(42, 0).sample(t, n - 4, out=buf[4:n])      # v4 (16-byte aligned)
        arv.Pcg32Stream(42, 0).sample(t, n - 1, out=buf[1:n])      # scalar stores
    # the lane-table headline kernel (512-thread CTAs, 59 KB tables) on the same sizes and alignments
    _native.call("arv_set_tuning", 5, 0)
    for t in (sub, lin):
        arv.Pcg32Stream(42, 0).sample(t, n, out=buf[:n])
        arv.Pcg32Stream(42, 0).sample(t, n - 4, out=buf[4:n])
    _native.call("arv_set_tuning", 5, 26)
    arv.Pcg32Stream(42, 0).sample("exact", 4096, out=buf[:4096])
    arv.Pcg32Stream(42, 0).sample_exact64(4096)
    arv.Pcg32Stream(42, 0).words(n)
    # lattice hook (whole 2^23 lattice, both evaluators)
    from paper_2012_09715_b200 import _device as dev

    c = torch.from_numpy(np.ascontiguousarray(sub.coeffs32)).cuda()
    lat = torch.empty(1 << 23, dtype=torch.float32, device="cuda")
    fast = torch.zeros(1, dtype=torch.int32, device="cuda")
    for mode in (0, 1, 2):
        _native.call("arv_lattice_subdyadic_f32", c.data_ptr(), 1, 16, 3, mode, lat.data_ptr(), fast.data_ptr(),
                     dev.stream_handle())
    # drop-in kernels, device and host buffers
    u = torch.rand(n, dtype=torch.float64, device="cuda").clamp_(1e-12, 1 - 1e-12)
    o = torch.empty_like(u)
    _kernels.dyadic_eval(lin.coeffs, u, o)
    _kernels.dyadic_eval32(lin.coeffs32, u.float(), o.float())
    _kernels.constant_eval(const.values, u, o)
    _kernels.dyadic_index(u, 15)
    _kernels.gaussian_inv_cdf(u, o)
    nc = arv.load_table("ncchi2_cir_k64_stacks")
    _kernels.ncchi2_eval(nc.eval_stacks, nc.nu, u, torch.full((1,), 7.5, dtype=torch.float64, device="cuda"), o)
    _kernels.ncchi2_eval(nc.eval_stacks, nc.nu, u, u * 100.0, o)
    uh = u.cpu().numpy()
    oh = np.empty_like(uh)
    _kernels.dyadic_eval(lin.coeffs, uh, oh)
    _kernels.ncchi2_eval(nc.eval_stacks, nc.nu, uh, uh * 50.0, oh)
    # ncchi2 quantile / cdf
    from paper_2012_09715_b200 import exact_dist

    exact_dist.ncchi2_inv_cdf_batch(u[:2048], nc.nu, u[:2048] * 300.0)
    # MLMC levels
    gbm, cir = arv.GbmParams(0.05, 0.2, 1.0, 1.0), arv.CirParams(0.5, 0.04, 0.2, 0.04, 1.0)
    np_ = (1 << 20) + 77 if big else 600_011  # > 2048 CTA partials: the atomic-ticket chunk finalize
    for scheme, proc, tab, lv in (("euler_maruyama", gbm, lin, 3), ("milstein", gbm, cub, 2),
                                  ("euler_maruyama", gbm, const, 1), ("cir_euler_truncated", cir, lin, 2),
                                  ("cir_milstein_truncated", cir, lin, 1), ("euler_maruyama", gbm, lin, 0)):
        sp = arv.LevelSpec(level=lv, scheme=scheme, process=proc, rv_source=tab, kind="four_way", n0=1)
        run_level(sp, arv.level_stream(42, lv), np_, want_paths=True)
        run_level(sp, arv.level_stream(42, lv), 1000, path_lo=333, path_count=500)
        run_level(sp, arv.level_stream(42, lv, generator="philox"), 5000)
    for lv, cnt in ((1, 3000), (5, 3000)):  # one-kernel (no sort), segmented
        sp = arv.LevelSpec(level=lv, scheme="cir_exact", process=cir, rv_source=nc, kind="four_way", n0=1)
        run_level(sp, arv.level_stream(42, lv), cnt, want_paths=True)
    _native.call("arv_set_tuning", 3, 0)  # CIR segments off: long level as one sorted kernel
    sp = arv.LevelSpec(level=4, scheme="cir_exact", process=cir, rv_source=nc, kind="four_way", n0=1)
    run_level(sp, arv.level_stream(42, 4), 2000, want_paths=True)
    torch.cuda.synchronize()
    print("sanitize workload done, launches:", _native.launch_count())


if __name__ == "__main__":
    main()

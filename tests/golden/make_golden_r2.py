"""Round-2 golden fixtures, made FROM THE REFERENCE ITSELF (and the pinned
oracle where the reference has no counterpart).

Runs only in the build container (needs /root/reference and oracle/_ref, see
make_golden.py).  Writes ``tests/golden/golden_r2.npz``,
``tests/golden/dropin_trace.npz`` + ``dropin_trace.json`` and adds keys to
``tests/golden/hashes.json``; nothing on the GPU box reads /root/reference.

  * sha256 of the full config-2 output (2^28 samples of the 16x8 sub-interval
    table from PCG32(42, 0)), from the oracle's fused generator (the
    sub-interval layout has no reference kernel; the oracle evaluator is pinned
    to the reference by degenerate equivalence, tests/test_oracle.py);
  * mlmc.simulate_cir_coupled(cir_exact) with the 64-KNOT table (BASELINE
    config 5) at levels 4 and 6, per path, PCG32 uniforms in the reference's
    own consumption order (mlmc.py:253-287);
  * mlmc.simulate_gbm_coupled with the CUBIC K15 table (dyadic_eval, m = 3),
    EM and Milstein, per path (mlmc.py:164-229);
  * a DROP-IN CALL TRACE: the reference's own sampler / mlmc / metrics code
    run with its plugin (`sampler.kernels`, _backend.py:14-24) wrapped in a
    recorder around the compiled reference kernels.  Every plugin call the
    reference makes -- arguments as the reference passes them (dtypes,
    shapes, scalar batches, shared / per-element lambda) and the outputs it
    gets back -- is stored.  tests/test_gpu_dropin.py replays the trace
    through paper_2012_09715_b200._kernels with the same numpy arguments: if
    every call returns the same bits, the reference's code computes the same
    results with the CUDA plugin swapped in (its code between plugin calls is
    deterministic numpy).  The reference package itself does not travel to
    the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
os.environ.setdefault("APPROXRV_BACKEND", "python")
sys.path.insert(0, "/root/reference/pkg/src")

import oracle  # noqa: E402
from approxrv import mlmc, sampler  # noqa: E402
from make_golden import (REF, TABLES, Pcg32UniformStream, mlmc_table, ref_const_table,  # noqa: E402
                         ref_ncchi2_table)


class Recorder:
    """Stands in for the reference's kernel module: forwards every call to the
    compiled reference kernels (oracle/_ref) and records it."""

    COMPILED = True
    NAMES = ("constant_eval", "dyadic_index", "dyadic_index32", "dyadic_eval", "dyadic_eval32", "ncchi2_eval")

    def __init__(self, inner):
        self.inner = inner
        self.calls = []

    def __getattr__(self, name):
        if name not in self.NAMES:
            raise AttributeError(name)
        fn = getattr(self.inner, name)

        def wrapped(*args):
            before = [np.array(a, copy=True) if isinstance(a, np.ndarray) else a for a in args]
            ret = fn(*args)
            after = [np.array(a, copy=True) if isinstance(a, np.ndarray) else None for a in args]
            self.calls.append((name, before, after, None if ret is None else np.array(ret, copy=True)))
            return ret

        return wrapped


def trace_reference_calls():
    rec = Recorder(REF)
    sampler.kernels = rec  # the reference's plugin slot (sampler.py:17)
    lin, cub = mlmc_table("dyadic_linear_k15"), mlmc_table("dyadic_cubic_k15")
    const = ref_const_table()
    nc64 = ref_ncchi2_table("ncchi2_cir_k64_stacks", "ncchi2_cir_k64_nu")
    labels = []

    def mark(label):
        labels.append((len(rec.calls), label))

    u = sampler.UniformStream(42, 3).uniforms(4099)
    mark("evaluate(constant)")
    sampler.evaluate(const, u)
    mark("evaluate(linear K15)")
    sampler.evaluate(lin, u)
    mark("evaluate(cubic K15)")
    sampler.evaluate(cub, u)
    mark("eval_dyadic(linear, float32)")
    sampler.eval_dyadic(lin, u, dtype=np.float32)
    mark("eval_dyadic(cubic, float32, out=)")
    sampler.eval_dyadic(cub, u.astype(np.float32), dtype=np.float32, out=np.empty(u.size, np.float32))
    mark("scalar calls")
    sampler.eval_dyadic(lin, 0.5)
    sampler.eval_dyadic(lin, 0.3)
    sampler.eval_constant(const, 0.73)
    sampler.dyadic_index(0.3)
    sampler.dyadic_index(2.0**-30, 15)
    mark("dyadic_index batches (f64 / f32)")
    sampler.dyadic_index(u, 15)
    sampler.dyadic_index(u.astype(np.float32), 15)
    mark("eval_ncchi2 shared and per-element lambda")
    sampler.eval_ncchi2(nc64, u[:1000], 7.5)
    sampler.eval_ncchi2(nc64, u[:1000], np.linspace(0.0, 400.0, 1000))
    mark("sample_coupled")
    sampler.sample_coupled(sampler.UniformStream(42, 9), lin, 2048)
    gbm = mlmc.GbmParams(mu=0.05, sigma=0.2, x0=1.0, t_end=1.0)
    mark("estimate_level_suite GBM EM level 3")
    spec = mlmc.LevelSpec(level=3, scheme="euler_maruyama", process=gbm, rv_source=lin, kind="four_way", n0=1)
    suite = mlmc.estimate_level_suite(spec, mlmc.level_stream(42, 3), 1000)
    mark("estimate_level_suite GBM Milstein call, cubic, level 2")
    spec = mlmc.LevelSpec(level=2, scheme="milstein", process=gbm, rv_source=cub, kind="four_way",
                          payoff="call", strike=1.0, n0=2)
    mlmc.estimate_level_suite(spec, mlmc.level_stream(42, 2), 500)
    mark("estimate_level_suite GBM constant table level 1")
    spec = mlmc.LevelSpec(level=1, scheme="euler_maruyama", process=gbm, rv_source=const, kind="four_way", n0=1)
    mlmc.estimate_level_suite(spec, mlmc.level_stream(42, 1), 700)
    cir = mlmc.CirParams(kappa=0.5, theta=0.04, sigma=0.2, x0=0.04, t_end=1.0)
    mark("simulate CIR exact 64 knots level 2")
    spec = mlmc.LevelSpec(level=2, scheme="cir_exact", process=cir, rv_source=nc64, kind="four_way", n0=1)
    mlmc.simulate(spec, mlmc.level_stream(42, 2), 300, sides="both")
    mark("simulate CIR truncated Euler level 3")
    spec = mlmc.LevelSpec(level=3, scheme="cir_euler_truncated", process=cir, rv_source=lin, kind="four_way", n0=1)
    mlmc.simulate(spec, mlmc.level_stream(42, 3), 400, sides="both")
    from approxrv import metrics

    mark("metrics.rmse_ncchi2 (Table 5 grid, small)")
    metrics.rmse_ncchi2([nc64], (1.0, 50.0), n_samples=1 << 10)

    arrays, manifest = {}, []
    for i, (name, before, after, ret) in enumerate(rec.calls):
        entry = {"name": name, "args": []}
        for j, (b, a) in enumerate(zip(before, after)):
            if isinstance(b, np.ndarray):
                arrays[f"c{i}_a{j}"] = b
                if a is not None and not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
                    arrays[f"c{i}_o{j}"] = a  # the argument was written (the caller's `out`)
                    entry["args"].append({"array": j, "out": True, "shape": list(b.shape), "dtype": str(b.dtype)})
                else:
                    entry["args"].append({"array": j, "out": False, "shape": list(b.shape), "dtype": str(b.dtype)})
            else:
                entry["args"].append({"scalar": b if not isinstance(b, np.generic) else b.item()})
        if ret is not None:
            arrays[f"c{i}_ret"] = ret
            entry["ret"] = True
        manifest.append(entry)
    summary = {k: [suite[k].mean, suite[k].variance] for k in ("two_way_exact", "two_way_approx", "four_way")}
    return arrays, {"calls": manifest, "labels": labels, "gbm_em_l3_suite": summary}


def main() -> None:
    g = {}
    with open(os.path.join(HERE, "hashes.json")) as fh:
        h = json.load(fh)

    # --------------------------------------- config 2, full size (2^28), oracle
    c = TABLES["subdyadic_linear_k16_s8"].astype(np.float32)
    n, ch = 1 << 28, 1 << 24
    hs = hashlib.sha256()
    with ThreadPoolExecutor(8) as ex:
        for a in ex.map(lambda off: oracle.pcg32_subdyadic_f32(42, 0, off, c, 3, ch), range(0, n, ch)):
            hs.update(a.tobytes())
    h["config2_subdyadic_f32_sha256_2^28"] = hs.hexdigest()

    # ------------------------------- CIR exact, 64-knot table, levels 4 and 6
    cir = mlmc.CirParams(kappa=0.5, theta=0.04, sigma=0.2, x0=0.04, t_end=1.0)
    nc64 = ref_ncchi2_table("ncchi2_cir_k64_stacks", "ncchi2_cir_k64_nu")
    cases = [(4, 1, 256), (6, 1, 128)]
    for level, n0, npaths in cases:
        spec = mlmc.LevelSpec(level=level, scheme="cir_exact", process=cir, rv_source=nc64, kind="four_way", n0=n0)
        b = mlmc.simulate(spec, Pcg32UniformStream(42, level << 32), npaths, sides="both")
        g[f"cir_exact64_l{level}_n{n0}"] = np.stack([b.p_fine_exact, b.p_fine_approx])
    h["cir_exact64_cases"] = [list(x) for x in cases]

    # ------------------------------------------------ GBM with the cubic table
    cub = mlmc_table("dyadic_cubic_k15")
    gbm = mlmc.GbmParams(mu=0.05, sigma=0.2, x0=1.0, t_end=1.0)
    cases = [("euler_maruyama", "identity", 0, 1), ("euler_maruyama", "identity", 3, 1),
             ("milstein", "call", 2, 2), ("euler_maruyama", "call", 5, 1)]
    for scheme, payoff, level, n0 in cases:
        spec = mlmc.LevelSpec(level=level, scheme=scheme, process=gbm, rv_source=cub, kind="four_way",
                              payoff=payoff, strike=1.0, n0=n0)
        b = mlmc.simulate(spec, Pcg32UniformStream(42, (level << 32) | 1), 512, sides="both")
        g[f"gbm_cubic_{scheme}_{payoff}_l{level}_n{n0}"] = np.stack(
            [b.p_fine_exact, b.p_coarse_exact, b.p_fine_approx, b.p_coarse_approx])
    h["gbm_cubic_cases"] = [list(x) for x in cases]

    # -------------------------------------------- sides semantics (mlmc.py:176-229)
    lin = mlmc_table("dyadic_linear_k15")
    spec = mlmc.LevelSpec(level=2, scheme="euler_maruyama", process=gbm, rv_source=lin, kind="four_way", n0=1)
    for sides in ("exact", "approx"):
        b = mlmc.simulate(spec, Pcg32UniformStream(42, 2 << 32), 256, sides=sides)
        present = [getattr(b, f) is not None for f in ("p_fine_exact", "p_coarse_exact", "p_fine_approx",
                                                        "p_coarse_approx")]
        h[f"sides_{sides}_present"] = present

    np.savez_compressed(os.path.join(HERE, "golden_r2.npz"), **g)
    with open(os.path.join(HERE, "hashes.json"), "w") as fh:
        json.dump(h, fh, indent=1)

    arrays, manifest = trace_reference_calls()
    np.savez_compressed(os.path.join(HERE, "dropin_trace.npz"), **arrays)
    with open(os.path.join(HERE, "dropin_trace.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("golden_r2:", sorted(g), "trace calls:", len(manifest["calls"]))


if __name__ == "__main__":
    main()

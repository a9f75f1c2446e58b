"""Generate the golden parity fixtures FROM THE REFERENCE ITSELF.

Runs only in the build container (needs /root/reference and the oracle's
``_ref`` build of the reference's Cython kernels: ``make -C oracle ref``).
Outputs ``tests/golden/golden.npz`` and ``tests/golden/hashes.json``, which
are committed; nothing on the GPU box reads /root/reference.

What is pinned (reference function -> fixture):
  * _kernels.constant_eval / dyadic_eval32 / dyadic_eval / dyadic_index(32) /
    ncchi2_eval (compiled Cython, oracle/_ref) on PCG32 lattice uniforms,
    random doubles and edge values;
  * exact_dist.gaussian_inv_cdf (AS241) on the same inputs;
  * mlmc.simulate_gbm_coupled and simulate_cir_coupled (cir_exact,
    cir_euler_truncated) per-path payoffs, with the reference's
    UniformStream swapped for a PCG32 stream that yields (w + 0.5) 2^-32 in
    the reference's own consumption order (one uniforms(n_paths) per step);
  * sha256 of the full config-1 output (2^24 samples) and of the K15 f32
    dyadic output (2^24), computed with the reference kernels.
PCG32 itself has no reference implementation; its words come from the
pure-Python restatement in oracle/oracle.py (pcg32_words_py), independent of
the C oracle, plus the published pcg32 demo sequence for (42, 54).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
os.environ.setdefault("APPROXRV_BACKEND", "python")
sys.path.insert(0, "/root/reference/pkg/src")

import oracle  # noqa: E402
from approxrv import exact_dist, mlmc  # noqa: E402

REF = oracle.load_ref_kernels()
assert REF is not None and REF.COMPILED, "build oracle/_ref first: make -C oracle ref"
TABLES = np.load(os.path.join(REPO, "paper_2012_09715_b200", "data", "tables.npz"))

EDGE_WORDS = np.array([0, 1, 511, 512, 1023, 0x003FFFFF, 0x00400000, 0x7FFFFDFF, 0x7FFFFE00, 0x7FFFFFFF,
                       0x80000000, 0x800001FF, 0x80000200, 0xFFFFFC00, 0xFFFFFDFF, 0xFFFFFE00, 0xFFFFFFFF,
                       0x00000200, 0x00000400, 0x00010000, 0xFFFF0000], dtype=np.uint32)
EDGE_F64 = np.array([0.5, 0.25, 0.3, 0.125, 2.0**-30, 2.0**-53, 1.0 - 2.0**-53, np.nextafter(0.5, 0),
                     np.nextafter(0.5, 1), 1e-300, 5e-324, 1e-310, 0.75, 0.999999, 1e-6])


class Pcg32UniformStream:
    """Drop-in for approxrv.sampler.UniformStream: PCG32 words -> (w+0.5) 2^-32."""

    def __init__(self, seed, stream_id):
        self.seed, self.stream_id, self.counter = seed, stream_id, 0

    def uniforms(self, n):
        w = oracle.pcg32_words(self.seed, self.stream_id, self.counter, n)
        self.counter += n
        return (w.astype(np.float64) + 0.5) * 2.0**-32


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    g = {}
    h = {}
    # ---------------------------------------------------------------- PCG32
    g["pcg_kat_42_54"] = oracle.pcg32_words_py(42, 54, 6)
    g["pcg_words_42_0"] = oracle.pcg32_words_py(42, 0, 4096)
    g["pcg_words_7_3_off"] = oracle.pcg32_words_py(7, 3, 300)[100:]  # offset 100 of (7, 3)

    # -------------------------------------------------- lattice uniforms f32
    w = np.concatenate([oracle.pcg32_words(42, 0, 0, 1 << 14), EDGE_WORDS])
    u32 = oracle.u32_to_f32(w)
    g["lattice_words"] = w
    g["lattice_u32"] = u32
    vals = TABLES["constant_q10_l1"]
    out = np.empty(w.size)
    REF.constant_eval(vals, u32.astype(np.float64), out)
    g["const_q10_out"] = out
    for name in ("dyadic_linear_k15", "dyadic_cubic_k15"):
        c32 = TABLES[name].astype(np.float32)
        o32 = np.empty_like(u32)
        REF.dyadic_eval32(c32, u32, o32)
        g[f"{name}_eval32_out"] = o32
    g["dyadic32_index_out"] = REF.dyadic_index32(u32, 15)

    # ------------------------------------------------------------ f64 inputs
    rng = np.random.default_rng(3)
    u64 = np.concatenate([rng.random(1 << 14), EDGE_F64])
    g["u64"] = u64
    for name in ("dyadic_linear_k15", "dyadic_cubic_k15"):
        o = np.empty_like(u64)
        REF.dyadic_eval(TABLES[name], u64, o)
        g[f"{name}_eval_out"] = o
    v = np.minimum(u64, 1.0 - u64)
    g["dyadic_index_cap15"] = REF.dyadic_index(u64, 15)
    g["dyadic_index_uncapped"] = REF.dyadic_index(v, 1 << 62)
    pow2 = 2.0 ** -np.arange(1, 40, dtype=np.float64)
    g["pow2"] = pow2
    g["pow2_index"] = REF.dyadic_index(pow2, 64)
    g["index32_probe"] = np.array([0.5, 0.26, 0.12, 2.0**-20, 1.0, 0.0, 2.0**-126, 1e-40], dtype=np.float32)
    g["index32_probe_out"] = REF.dyadic_index32(g["index32_probe"], 15)
    g["constant_u64_out"] = np.empty_like(u64)
    REF.constant_eval(vals, u64, g["constant_u64_out"])

    # ----------------------------------------------------------------- AS241
    tails = np.concatenate([10.0 ** -np.arange(1.0, 300.0, 7.0), 1.0 - 10.0 ** -np.arange(1.0, 16.0)])
    ua = np.concatenate([u64[(u64 > 0) & (u64 < 1)], tails, (w.astype(np.float64) + 0.5) * 2.0**-32])
    g["as241_u"] = ua
    g["as241_out"] = exact_dist.gaussian_inv_cdf(ua)

    # ---------------------------------------------------------------- ncchi2
    st = TABLES["ncchi2_cir_k64_stacks"]
    nu = float(TABLES["ncchi2_cir_k64_nu"])
    un = rng.random(4096)
    lam = rng.random(4096) * 300.0
    lam[:8] = [0.0, 1e-12, 1e12, 7.5, 250.0, 3.0, 1e-3, 1e3]
    g["ncchi2_u"], g["ncchi2_lam"] = un, lam
    o = np.empty_like(un)
    REF.ncchi2_eval(st, nu, un, lam, o)
    g["ncchi2_k64_perelem_out"] = o
    o = np.empty_like(un)
    REF.ncchi2_eval(st, nu, un, np.full(1, 7.5), o)
    g["ncchi2_k64_shared_out"] = o

    # ------------------------------------------------------------------ GBM
    lin = mlmc_table("dyadic_linear_k15")
    gbm = mlmc.GbmParams(mu=0.05, sigma=0.2, x0=1.0, t_end=1.0)
    cases = []
    for scheme in ("euler_maruyama", "milstein"):
        for payoff in ("identity", "call"):
            for level, n0 in ((0, 1), (1, 1), (2, 1), (4, 1), (3, 2), (0, 3)):
                cases.append((scheme, payoff, level, n0))
    n_paths = 512
    for scheme, payoff, level, n0 in cases:
        spec = mlmc.LevelSpec(level=level, scheme=scheme, process=gbm, rv_source=lin, kind="four_way",
                              payoff=payoff, strike=1.0, n0=n0)
        stream = Pcg32UniformStream(42, (level << 32) | 0)
        b = mlmc.simulate(spec, stream, n_paths, sides="both")
        key = f"gbm_{scheme}_{payoff}_l{level}_n{n0}"
        g[key] = np.stack([b.p_fine_exact, b.p_coarse_exact, b.p_fine_approx, b.p_coarse_approx])
    h["gbm_cases"] = [list(c) for c in cases]
    h["gbm_n_paths"] = n_paths

    # ------------------------------- Philox replay (the reference's own streams)
    # UniformStream itself (no substitution): uniforms, evaluate() and the GBM
    # pilot exactly as the reference runs them with level_stream(seed, level).
    from approxrv import sampler as ref_sampler

    g["philox_uniforms_5_3_c13"] = ref_sampler.UniformStream(5, (3 << 32) | 1, counter=13).uniforms(4099)
    g["philox_words_42_7"] = ref_sampler.UniformStream(42, 7).raw_words(64)
    uu = ref_sampler.UniformStream(42, 9).uniforms(8192)
    g["philox_eval_dyadic_lin"] = ref_sampler.evaluate(lin, uu)
    g["philox_eval_const"] = ref_sampler.evaluate(ref_const_table(), uu)
    g["philox_eval_exact"] = exact_dist.gaussian_inv_cdf(uu)
    ph_cases = []
    for scheme, payoff, level, n0 in (("euler_maruyama", "identity", 3, 1), ("milstein", "call", 2, 2),
                                      ("euler_maruyama", "identity", 0, 1), ("euler_maruyama", "identity", 5, 1)):
        spec = mlmc.LevelSpec(level=level, scheme=scheme, process=gbm, rv_source=lin, kind="four_way",
                              payoff=payoff, strike=1.0, n0=n0)
        b = mlmc.simulate(spec, mlmc.level_stream(42, level), 1000, sides="both")
        g[f"philox_gbm_{scheme}_{payoff}_l{level}_n{n0}"] = np.stack(
            [b.p_fine_exact, b.p_coarse_exact, b.p_fine_approx, b.p_coarse_approx])
        suite = mlmc.estimate_level_suite(spec, mlmc.level_stream(42, level), 1000)
        g[f"philox_suite_{scheme}_{payoff}_l{level}_n{n0}"] = np.array(
            [[suite[k].mean, suite[k].variance] for k in ("two_way_exact", "two_way_approx", "four_way")])
        ph_cases.append([scheme, payoff, level, n0])
    h["philox_gbm_cases"] = ph_cases

    # ------------------------------------------------------------------ CIR
    cir = mlmc.CirParams(kappa=0.5, theta=0.04, sigma=0.2, x0=0.04, t_end=1.0)
    from approxrv.tables import NcChi2Table  # noqa: F401
    tab = ref_ncchi2_table("ncchi2_cir_k16_stacks", "ncchi2_cir_k16_nu")
    cir_cases = [(0, 1), (1, 1), (2, 1)]
    for level, n0 in cir_cases:
        spec = mlmc.LevelSpec(level=level, scheme="cir_exact", process=cir, rv_source=tab, kind="four_way", n0=n0)
        b = mlmc.simulate(spec, Pcg32UniformStream(42, (level << 32)), 256, sides="both")
        g[f"cir_exact_l{level}_n{n0}"] = np.stack([b.p_fine_exact, b.p_fine_approx])
    h["cir_exact_cases"] = [list(c) for c in cir_cases]
    for level, n0 in ((0, 1), (3, 1), (2, 2)):
        spec = mlmc.LevelSpec(level=level, scheme="cir_euler_truncated", process=cir, rv_source=lin,
                              kind="four_way", n0=n0)
        b = mlmc.simulate(spec, Pcg32UniformStream(42, (level << 32) | 5), 512, sides="both")
        g[f"cir_euler_l{level}_n{n0}"] = np.stack([b.p_fine_exact, b.p_coarse_exact, b.p_fine_approx,
                                                  b.p_coarse_approx])
    h["cir_euler_cases"] = [[0, 1], [3, 1], [2, 2]]

    # ------------------------------------------------ full-size output hashes
    n = 1 << 24
    chunk = 1 << 22
    hc, hd = hashlib.sha256(), hashlib.sha256()
    c32 = TABLES["dyadic_linear_k15"].astype(np.float32)
    for off in range(0, n, chunk):
        uu = oracle.u32_to_f32(oracle.pcg32_words(42, 0, off, chunk))
        oc = np.empty(chunk)
        REF.constant_eval(vals, uu.astype(np.float64), oc)
        hc.update(oc.astype(np.float32).tobytes())
        od = np.empty_like(uu)
        REF.dyadic_eval32(c32, uu, od)
        hd.update(od.tobytes())
    h["config1_const_q10_f32_sha256_2^24"] = hc.hexdigest()
    h["dyadic_linear_k15_f32_sha256_2^24"] = hd.hexdigest()

    # -------------------------------------- ARVT files written by the reference
    from approxrv import tableio

    arvt = os.path.join(HERE, "arvt")
    os.makedirs(arvt, exist_ok=True)
    nc16 = ref_ncchi2_table("ncchi2_cir_k16_stacks", "ncchi2_cir_k16_nu")
    cubic = mlmc_table("dyadic_cubic_k15")
    for name, tab in (("constant_q10", ref_const_table()), ("dyadic_linear_k15", lin), ("dyadic_cubic_k15", cubic),
                      ("ncchi2_cir_k16", nc16)):
        tableio.export_table(tab, os.path.join(arvt, f"{name}.arvt"))
        tableio.export_table(tab, os.path.join(arvt, f"{name}.txt"), format="text")

    # ------------------------------------- Table-5 style RMSE grid (metrics.py:324-350)
    from approxrv import metrics

    grid = metrics.rmse_ncchi2([ref_ncchi2_table("ncchi2_nu1_k16_stacks", "ncchi2_nu1_k16_nu"), nc16_ref()],
                               (1.0, 5.0, 10.0, 50.0, 100.0, 200.0), n_samples=1 << 14)
    g["rmse_grid_values"] = grid.values
    g["rmse_grid_lambdas"] = np.array(grid.lambdas)

    # ------------------------------- the reference's MLMC experiment driver
    from approxrv import cli

    exp_cfg = {"process": "gbm", "scheme": "euler_maruyama", "seed": "42", "pilot": "4000", "epsilon": "0.01",
               "levels": "0:4", "sources": "exact,linear:15", "n0": "2"}
    cli.run_experiment(dict(exp_cfg), os.path.join(HERE, "experiment_ref"))
    with open(os.path.join(HERE, "experiment_ref", "config.json"), "w") as fh:
        json.dump(exp_cfg, fh, indent=1)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    with open(os.path.join(HERE, "hashes.json"), "w") as fh:
        json.dump(h, fh, indent=1)
    print("wrote", len(g), "arrays;", h)


def mlmc_table(name):
    from approxrv.tables import DyadicPolyTable

    c = TABLES[name]
    return DyadicPolyTable(degree=c.shape[0] - 1, n_intervals=c.shape[1] - 1, coeffs=c)


def nc16_ref():
    return ref_ncchi2_table("ncchi2_cir_k16_stacks", "ncchi2_cir_k16_nu")


def ref_const_table():
    from approxrv.tables import ConstantTable

    return ConstantTable(q=10, values=TABLES["constant_q10_l1"], construction="l1")


def ref_ncchi2_table(stacks_key, nu_key):
    """Rebuild a reference NcChi2Table from the shipped stacks (upper at 0, lower at 1)."""
    from approxrv.tables import DyadicPolyTable, NcChi2Table

    s = TABLES[stacks_key]
    nu = float(TABLES[nu_key])
    m, k = s.shape[2] - 1, s.shape[3] - 1
    lower = tuple(DyadicPolyTable(m, k, s[1, j]) for j in range(s.shape[1]))
    upper = tuple(DyadicPolyTable(m, k, s[0, j]) for j in range(s.shape[1]))
    t = NcChi2Table(nu=nu, n_knots=s.shape[1], degree=m, n_intervals=k, lower=lower, upper=upper)
    assert np.array_equal(t.eval_stacks, s)
    return t


if __name__ == "__main__":
    main()

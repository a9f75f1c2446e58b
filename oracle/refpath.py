"""CPU baselines of the reference's host paths (BENCH INFRASTRUCTURE ONLY).

Used by bench.py's cpu_baseline / --impl reference legs and nowhere in the
product.  Each worker runs in its own process (the reference's Cython
kernels hold the GIL; numpy/scipy loops are single-threaded), one per host
core, on disjoint streams / path ranges, as SURVEY.md §8(d) "CPU baseline"
asks ("all cores via a process pool, with N/cores per process on disjoint
stream ids").

* ``sampler_path``: the reference's own sampling path, sampler.py:48-62 +
  :144-172 -- ``UniformStream.uniforms`` (numpy's Philox-4x64 bit generator
  keyed [seed, stream_id], u = ((w >> 11) + 0.5) 2^-53; numpy is the
  reference's own dependency) then ``eval_dyadic(table, u, float32)``: the
  f64 -> f32 cast and the reference's compiled ``dyadic_eval32``
  (oracle/_ref, _kernels.pyx:76-93).  Generation included.
* ``gbm_level``: the C restatement of ``simulate_gbm_coupled``
  (oracle.c orc_gbm_paths, mlmc.py:164-229; pinned per path to the
  reference in tests/test_oracle.py) plus the per-path differences and
  their moments (mlmc.py:341-411).
* ``cir_exact_level``: the numpy/scipy restatement of
  ``simulate_cir_coupled(cir_exact)`` (oracle/cir.py, mlmc.py:253-287,
  exact_dist.py:381-461 with scipy's CDFLIB ``chndtr``).
"""

from __future__ import annotations

import os
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_TABLES = os.path.join(os.path.dirname(_HERE), "paper_2012_09715_b200", "data", "tables.npz")


def _tables():
    with np.load(_TABLES) as z:
        return {k: z[k] for k in z.files}


def sampler_path(args):
    """(samples, seconds): UniformStream(seed, sid).uniforms + eval_dyadic f32, in chunks."""
    from numpy.random import Philox

    from . import oracle

    seed, sid, n, chunk = args
    ref = oracle.load_ref_kernels()
    c32 = _tables()["dyadic_linear_k15"].astype(np.float32)
    key = np.array([seed, sid], dtype=np.uint64)
    out = np.empty(chunk, np.float32)
    t0 = time.perf_counter()
    done = 0
    while done < n:
        m = min(chunk, n - done)
        block, off = divmod(done, 4)  # sampler.py:51-56
        w = Philox(key=key, counter=block).random_raw(off + m)[off:]
        u = ((w >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0**-53  # sampler.py:62
        u32 = np.ascontiguousarray(u, dtype=np.float32)  # sampler.py:165
        ref.dyadic_eval32(c32, u32, out[:m])
        done += m
    return n, time.perf_counter() - t0


def gbm_level(args):
    """(path_steps, seconds): coupled GBM EM paths (both sides) + the three
    difference kinds' moments, config 4 parameters, K15 linear table."""
    from . import oracle

    level, n_paths, path_lo, path_hi = args
    lin = _tables()["dyadic_linear_k15"]
    t0 = time.perf_counter()
    fe, ce, fa, ca = oracle.gbm_paths(mu=0.05, sigma=0.2, x0=1.0, t_end=1.0, level=level, n0=1, milstein=False,
                                      payoff_call=False, strike=1.0, coeffs=lin, seed=42, seq=level << 32,
                                      n_paths=n_paths, path_lo=path_lo, path_hi=path_hi)
    for d in (fe - ce, fa - ca, fe - ce - fa + ca):  # mlmc.py:341-353, 356-411
        float(d.mean()), float(d.var(ddof=1))
    return (path_hi - path_lo) << level, time.perf_counter() - t0


def cir_exact_level(args):
    """(transitions, seconds): coupled CIR exact paths, config 5 parameters, 64-knot table."""
    from . import cir

    level, n_paths, seed = args
    t = _tables()
    t0 = time.perf_counter()
    xe, xa, worst = cir.cir_exact_paths(kappa=0.5, theta=0.04, sigma=0.2, x0=0.04, t_end=1.0, level=level, n0=1,
                                        stacks=t["ncchi2_cir_k64_stacks"], nu_table=float(t["ncchi2_cir_k64_nu"]),
                                        seed=seed, seq=level << 32, n_paths=n_paths)
    float((xe - xa).var(ddof=1))
    return n_paths << level, time.perf_counter() - t0


def run_pool(fn, jobs, procs: int):
    """Run jobs on `procs` spawned processes; (units, wall seconds)."""
    import multiprocessing as mp

    with mp.get_context("spawn").Pool(procs) as pool:
        pool.map(_noop, range(procs))  # start-up (imports) outside the timing
        t0 = time.perf_counter()
        res = pool.map(fn, jobs)
        wall = time.perf_counter() - t0
    return sum(r[0] for r in res), wall


def _noop(_):
    from . import oracle  # noqa: F401
    from . import cir  # noqa: F401

    return 0

"""C-ABI library and host-side logic, CPU only (no kernel is launched).

* libarv_b200.so loads and exports every entry point include/*.h declares;
* argument validation happens before any CUDA call and maps onto the
  reference exception hierarchy (errors.py:9-42);
* the host mirror of the reference API (tables, LevelSpec, allocation,
  speed-up accounting, shard ranges, triple merges) behaves like mlmc.py.
"""

import ctypes
import glob
import math
import os
import re
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    names = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        txt = open(h).read()
        names |= set(re.findall(r"ARV_API\s+[\w\s\*]+?\b(arv_\w+)\s*\(", txt))
    return names


@pytest.fixture(scope="module")
def nat():
    from paper_2012_09715_b200 import _native

    return _native


def test_header_declares_entry_points():
    names = header_symbols()
    assert len(names) >= 25
    for must in ("arv_constant_eval", "arv_dyadic_index", "arv_dyadic_index32", "arv_dyadic_eval",
                 "arv_dyadic_eval32", "arv_ncchi2_eval", "arv_pcg32_subdyadic_f32", "arv_mlmc_gaussian_level"):
        assert must in names


def test_library_exports_every_declared_symbol(nat):
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH], capture_output=True, text=True, check=True)
    exported = {ln.split()[-1] for ln in out.stdout.splitlines() if " T " in ln}
    missing = header_symbols() - exported
    assert not missing, missing
    assert set(nat.EXPORTED_SYMBOLS) == header_symbols()
    for name in header_symbols():
        assert isinstance(getattr(nat.lib, name), ctypes._CFuncPtr)


def test_library_is_sm100a_and_in_tree(nat):
    assert nat.LIB_PATH.startswith(os.path.join(REPO, "paper_2012_09715_b200"))
    out = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True, text=True)
    if out.returncode == 0:
        assert "sm_100a" in out.stdout


def test_abi_version_and_no_launch_on_import(nat):
    assert nat.lib.arv_abi_version() == 1
    assert nat.launch_count() == 0


class TestValidationBeforeCuda:
    """Entry points reject bad arguments with a code and message, without CUDA."""

    def test_codes(self, nat):
        from paper_2012_09715_b200 import errors

        with pytest.raises(errors.ConfigError, match="q must be in"):
            nat.call("arv_pcg32_constant_f32", 42, 0, 0, None, 30, None, 16, None)
        with pytest.raises(errors.ConfigError, match="degree"):
            nat.call("arv_pcg32_subdyadic_f32", 42, 0, 0, None, 7, 16, 3, None, 16, None)
        with pytest.raises(errors.ConfigError, match="sub_bits"):
            nat.call("arv_subdyadic_eval32", None, 1, 16, 9, None, None, 16, None)
        with pytest.raises(errors.ConfigError, match="per-element lambda"):
            nat.call("arv_ncchi2_eval", None, 64, 1, 16, 2.0, None, None, 3, None, 5, None)
        with pytest.raises(errors.DomainError):
            nat.call("arv_ncchi2_inv_cdf", None, None, 1, -1.0, None, None, None, 4, None)
        with pytest.raises(errors.ConfigError, match="group must be"):
            nat.call("arv_set_tuning", 1, 5)
        with pytest.raises(errors.ConfigError, match="lane_min_n"):
            nat.call("arv_set_tuning", 5, 41)
        nat.call("arv_set_tuning", 5, 26)
        assert nat.launch_count() == 0

    def test_zero_length_is_a_noop(self, nat):
        for name, args in (("arv_constant_eval", (None, 4, None, None, 0, None)),
                           ("arv_dyadic_index", (None, 0, 15, None, None)),
                           ("arv_pcg32_words", (1, 2, 3, None, 0, None)),
                           ("arv_pcg32_subdyadic_f32", (1, 2, 3, None, 1, 16, 3, None, 0, None))):
            nat.call(name, *args)
        assert nat.launch_count() == 0

    def test_level_spec_validation(self, nat):
        from paper_2012_09715_b200 import errors

        s = nat.LevelSpec()
        s.a, s.b, s.x0, s.t_end, s.level, s.n0, s.scheme = 0.05, 0.2, 1.0, 1.0, 3, 1, nat.SCHEME_EM
        s.n_paths_total, s.path_lo, s.path_count = 100, 50, 100  # range past the end
        with pytest.raises(errors.ConfigError, match="path range"):
            nat.call("arv_mlmc_gaussian_level", ctypes.byref(s), None, 1, 16, None, None, None, 0, None)
        s.path_lo, s.path_count, s.scheme = 0, 100, nat.SCHEME_CIR_EXACT
        with pytest.raises(errors.ConfigError, match="cannot run scheme"):
            nat.call("arv_mlmc_gaussian_level", ctypes.byref(s), None, 1, 16, None, None, None, 0, None)
        s.scheme = nat.SCHEME_EM
        with pytest.raises(errors.ConfigError, match="workspace"):
            nat.call("arv_mlmc_gaussian_level", ctypes.byref(s), None, 1, 16, None, None, None, 0, None)
        parts = (1 << 22) // 256 * 15 * 8
        assert nat.lib.arv_mlmc_workspace_bytes(1 << 22) >= parts  # + chunked-finalize scratch
        s.sides = 7
        with pytest.raises(errors.ConfigError, match="sides"):
            nat.call("arv_mlmc_gaussian_level", ctypes.byref(s), None, 1, 16, None, None, None, 1 << 30, None)

    def test_host_buffer_entry_points_validate_first(self, nat):
        """arv_host_* (host numpy buffers) reject bad lengths / pointers and treat
        n = 0 as a no-op before touching CUDA (no pipeline is created)."""
        from paper_2012_09715_b200 import errors

        u = np.zeros(4)
        with pytest.raises(errors.ConfigError, match="negative length"):
            nat.call("arv_host_dyadic_eval", None, 1, 16, u.ctypes.data, u.ctypes.data, -1, None)
        with pytest.raises(errors.ConfigError, match="null host pointer"):
            nat.call("arv_host_dyadic_eval", None, 1, 16, None, u.ctypes.data, 4, None)
        with pytest.raises(errors.ConfigError, match="1 or n elements"):
            nat.call("arv_host_ncchi2_eval", None, 64, 1, 16, 2.0, u.ctypes.data, u.ctypes.data, 3, u.ctypes.data,
                     4, None)
        for name, args in (("arv_host_dyadic_eval32", (None, 1, 16, None, None, 0, None)),
                           ("arv_host_constant_eval", (None, 1024, None, None, 0, None)),
                           ("arv_host_dyadic_index", (None, 0, 15, None, None)),
                           ("arv_host_gaussian_inv_cdf", (None, None, 0, None))):
            nat.call(name, *args)
        assert nat.launch_count() == 0


class TestHostMirror:
    def test_tables(self):
        import paper_2012_09715_b200 as arv

        const = arv.load_table("constant_q10_l1")
        assert const.q == 10 and const.values.shape == (1024,) and not const.values.flags.writeable
        v = const.values
        assert np.all(np.diff(v) > 0) and np.array_equal(v[:512], -v[::-1][:512])
        lin = arv.load_table("dyadic_linear_k15")
        assert lin.coeffs.shape == (2, 16) and np.all(lin.coeffs[:, 0] == 0)
        assert lin.interval_bounds(1) == (0.25, 0.5) and lin.interval_bounds(15) == (0.0, 2.0**-15)
        sub = arv.load_table("subdyadic_linear_k16_s8")
        assert (sub.degree, sub.n_octaves, sub.sub_bits) == (1, 16, 3)
        assert np.all(sub.coeffs[:, 15, :] == sub.coeffs[:, 15, :1])  # singular octave replicated
        nc = arv.load_table("ncchi2_cir_k64_stacks")
        assert nc.n_knots == 64 and nc.eval_stacks.shape == (2, 64, 2, 16)
        assert nc.nu == 4.0 * 0.5 * 0.04 / 0.2**2  # 1.9999999999999996, cli.py:273
        with pytest.raises(arv.ConfigError):
            arv.ConstantTable(q=0, values=[1.0])
        with pytest.raises(arv.ConfigError):
            arv.DyadicPolyTable(degree=7, n_intervals=15, coeffs=np.zeros((8, 16)))
        with pytest.raises(arv.ConfigError):
            arv.SubDyadicTable(degree=1, n_octaves=16, sub_bits=6, coeffs=np.zeros((2, 16, 64)))

    def test_subdyadic_from_reference_layout(self):
        import paper_2012_09715_b200 as arv

        lin = arv.load_table("dyadic_linear_k15")
        t = arv.SubDyadicTable.from_dyadic(lin, sub_bits=3)
        assert t.coeffs.shape == (2, 15, 8)
        assert np.array_equal(t.coeffs[:, :, 5], lin.coeffs[:, 1:])

    def test_level_spec_validation_mirrors_reference(self):
        import paper_2012_09715_b200 as arv

        gbm = arv.GbmParams(0.05, 0.2, 1.0, 1.0)
        cir = arv.CirParams(0.5, 1.0, 1.0, 1.0, 1.0)
        lin = arv.load_table("dyadic_linear_k15")
        nc = arv.load_table("ncchi2_nu1_k16_stacks")
        spec = arv.LevelSpec(level=3, scheme="euler_maruyama", process=gbm, rv_source=lin, kind="four_way")
        assert spec.n_steps_fine == 16 and spec.dt_fine == 1.0 / 16.0
        bad = [
            dict(level=0, scheme="euler_maruyama", process=gbm, kind="four_way"),
            dict(level=0, scheme="cir_exact", process=gbm, rv_source=nc),
            dict(level=0, scheme="euler_maruyama", process=gbm, rv_source=nc, kind="two_way"),
            dict(level=0, scheme="cir_exact", process=cir, rv_source=lin, kind="two_way"),
            dict(level=-1, scheme="euler_maruyama", process=gbm),
            dict(level=0, scheme="nope", process=gbm),
            dict(level=0, scheme="euler_maruyama", process=gbm, n0=0),
        ]
        for kw in bad:
            with pytest.raises(arv.ConfigError):
                arv.LevelSpec(**kw)
        with pytest.raises(arv.ConfigError):
            arv.GbmParams(mu=0.0, sigma=0.0, x0=1.0, t_end=1.0)
        assert cir.feller_satisfied
        assert not arv.CirParams(0.5, 0.04, 0.2, 0.04, 1.0).feller_satisfied  # 1 ulp short (SURVEY §7 vii)

    def test_level_stream_ids(self):
        import paper_2012_09715_b200 as arv

        s = arv.level_stream(42, 5, 3)
        assert (s.seed, s.stream_id, s.counter) == (42, (5 << 32) | 3, 0)
        with pytest.raises(arv.ConfigError):
            arv.Pcg32Stream(seed=-1)

    @pytest.mark.parametrize("n,world", [(1 << 28, 8), (1000003, 3), (7, 4), (0, 2)])
    def test_shard_range(self, n, world):
        import paper_2012_09715_b200 as arv

        ranges = [arv.shard_range(n, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
            assert a1 == b0 and a0 <= a1
        assert all(lo % 8 == 0 or lo == n for lo, _ in ranges)

    def test_merge_triples_matches_two_pass(self):
        from paper_2012_09715_b200.mlmc import merge_triples

        rng = np.random.default_rng(0)
        x = rng.normal(1.05, 0.2, 10007)
        parts = np.array_split(x, 13)
        tri = np.array([[p.size, p.mean(), ((p - p.mean()) ** 2).sum()] for p in parts])
        n, mean, m2 = merge_triples(tri)
        assert n == x.size
        assert mean == pytest.approx(x.mean(), rel=1e-14)
        assert m2 / (n - 1) == pytest.approx(x.var(ddof=1), rel=1e-12)


class TestAllocationMirror:
    """Closed-form checks of test_mlmc.py:182-261 against the host mirror."""

    def _stats(self, pairs):
        import paper_2012_09715_b200 as arv

        return [arv.LevelStats(level=i, kind="two_way", mean=0.0, variance=v, n_paths=100,
                               cost_per_path_seconds=c, cost_per_path_draws=c) for i, (v, c) in enumerate(pairs)]

    def test_single_level(self):
        import paper_2012_09715_b200 as arv

        alloc = arv.optimal_allocation(self._stats([(1.0, 1.0)]), epsilon=math.sqrt(2.0))
        assert alloc.predicted_cost == pytest.approx(1.0) and alloc.n_paths == [1]

    def test_two_level_ratio(self):
        import paper_2012_09715_b200 as arv

        eps = math.sqrt(2.0)
        alloc = arv.optimal_allocation(self._stats([(4.0, 1.0), (1.0, 4.0)]), eps)
        total = 2.0 * eps**-2 * 4.0**2
        assert alloc.predicted_cost == pytest.approx(total)
        m0 = eps**-1 * math.sqrt(2.0 * total * 4.0)
        m1 = eps**-1 * math.sqrt(2.0 * total / 4.0)
        assert alloc.n_paths == [math.ceil(m0), math.ceil(m1)]

    def test_budget(self):
        import paper_2012_09715_b200 as arv

        alloc = arv.optimal_allocation(self._stats([(2.0, 1.0), (0.5, 3.0), (0.1, 10.0)]), epsilon=0.05)
        assert alloc.variance_budget_used <= 0.05**2 / 2.0 + 1e-15

    def test_speedup_formulas(self):
        from paper_2012_09715_b200.mlmc import speedup_row

        def suite(gap):
            import paper_2012_09715_b200 as arv

            mk = lambda v: arv.LevelStats(2, "two_way", 0.0, v, 100, 1.0, 1.0)  # noqa: E731
            return {"two_way_exact": mk(1.0), "four_way": mk(2.0**gap)}

        row = speedup_row("linear", [suite(-14.0)], cost_ratio=7.0)
        assert row.efficiency == pytest.approx(0.957, abs=2e-3)
        assert row.speedup == pytest.approx(6.70, abs=0.02)

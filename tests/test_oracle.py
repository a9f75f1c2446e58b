"""Pin the CPU oracle against the reference's own outputs (tests/golden).

CPU only.  Every comparison of integer/index/f32 lattice work is bit-exact;
AS241 tails (numpy log vs libm log) use a stated ulp-level tolerance.
"""

import hashlib

import numpy as np
import pytest

# Published pcg32 demo (pcg-c-basic, pcg32_srandom_r(42, 54)): first outputs.
PCG32_DEMO_42_54 = [0xA15C02B7, 0x7B47F409, 0xBA1D3330, 0x83D2F293, 0xBFA4784B, 0xCBED606E]


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


class TestPcg32:
    def test_published_demo_sequence(self, orc, golden):
        assert list(orc.pcg32_words(42, 54, 0, 6)) == PCG32_DEMO_42_54
        assert list(golden["pcg_kat_42_54"]) == PCG32_DEMO_42_54

    def test_c_matches_pure_python(self, orc, golden):
        assert np.array_equal(orc.pcg32_words(42, 0, 0, 4096), golden["pcg_words_42_0"])
        assert np.array_equal(orc.pcg32_words(7, 3, 100, 200), golden["pcg_words_7_3_off"])

    @pytest.mark.parametrize("offset", [0, 1, 3, 4, 1000, 123457])
    def test_jump_ahead_is_offset(self, orc, offset):
        full = orc.pcg32_words(9, 11, 0, offset + 64)
        assert np.array_equal(orc.pcg32_words(9, 11, offset, 64), full[offset:])

    def test_jump_composition(self, orc):
        _, inc = orc.pcg32_seed(1, 2)
        a1, c1 = orc.lcg_jump(12345, inc)
        a2, c2 = orc.lcg_jump(67890, inc)
        a, c = orc.lcg_jump(12345 + 67890, inc)
        m = (1 << 64) - 1
        assert a == (a2 * a1) & m and c == (a2 * c1 + c2) & m

    def test_f64_uniform_integer_domain(self, orc):
        """one_plus_u32 (arv_common.cuh): D = 1 + u assembled from the word's bits,
        u - 1/2 = D - 3/2, and AS241's |u - 1/2| <= 0.425 / u > 1/2 as integer
        compares on w -- all equal to the reference's f64 arithmetic."""
        lo, span = 322122547, 3650722201
        edges = [0, 1, 2**31 - 1, 2**31, 2**31 + 1, 2**32 - 1, lo - 1, lo, lo + 1, lo + span - 1, lo + span,
                 lo + span + 1]
        rng = np.random.default_rng(11)
        w = np.concatenate([np.array(edges, dtype=np.uint64), rng.integers(0, 2**32, 200_000, dtype=np.uint64)])
        w = w.astype(np.uint32)
        u = orc.u32_to_f64(w)  # (w + 1/2) 2^-32, the reference-order f64 map
        d_bits = (np.uint64(0x3FF00000) | (w.astype(np.uint64) >> np.uint64(12))) << np.uint64(32) | \
            ((w.astype(np.uint64) << np.uint64(20)) & np.uint64(0xFFFFFFFF)) | np.uint64(0x80000)
        D = d_bits.view(np.float64)
        assert np.array_equal(bits(D - 1.0), bits(u))
        assert np.array_equal(bits(D - 1.5), bits(u - 0.5))
        assert np.array_equal(bits(2.0 - D), bits(1.0 - u))
        central = ((w.astype(np.int64) - lo) % 2**32) <= span
        assert np.array_equal(central, np.abs(u - 0.5) <= 0.425)
        assert np.array_equal(w >= np.uint32(2**31), u > 0.5)

    def test_lattice_mapping(self, orc, golden):
        u = orc.u32_to_f32(golden["lattice_words"])
        assert np.array_equal(bits(u), bits(golden["lattice_u32"]))
        assert u.min() > 0 and u.max() < 1 and not np.any(u == 0.5)
        k = golden["lattice_words"] >> np.uint32(9)
        assert np.array_equal(u.astype(np.float64), (k.astype(np.float64) + 0.5) * 2.0**-23)


class TestPhilox:
    """The reference's own uniform source (UniformStream = numpy Philox-4x64-10)."""

    def test_words_match_reference_stream(self, orc, golden):
        assert np.array_equal(orc.philox_words(42, 7, 0, 64), golden["philox_words_42_7"])

    def test_words_match_numpy_philox(self, orc):
        from numpy.random import Philox

        ref = Philox(key=np.array([3, 2**63 + 5], dtype=np.uint64), counter=0).random_raw(1003)
        assert np.array_equal(orc.philox_words(3, 2**63 + 5, 0, 1003), ref)
        assert np.array_equal(orc.philox_words(3, 2**63 + 5, 17, 986), ref[17:])

    def test_uniforms_match_reference_stream(self, orc, golden):
        u = orc.philox_uniforms(5, (3 << 32) | 1, 13, 4099)
        assert np.array_equal(u, golden["philox_uniforms_5_3_c13"])


class TestPluginKernels:
    def test_constant_eval(self, orc, golden, tables_npz):
        v = tables_npz["constant_q10_l1"]
        out = orc.constant_eval(v, golden["lattice_u32"].astype(np.float64))
        assert np.array_equal(bits(out), bits(golden["const_q10_out"]))
        out = orc.constant_eval(v, golden["u64"])
        assert np.array_equal(bits(out), bits(golden["constant_u64_out"]))

    def test_constant_index_is_top_bits(self, golden, tables_npz):
        v = tables_npz["constant_q10_l1"]
        w = golden["lattice_words"]
        assert np.array_equal(golden["const_q10_out"], v[w >> np.uint32(22)])

    @pytest.mark.parametrize("name", ["dyadic_linear_k15", "dyadic_cubic_k15"])
    def test_dyadic_eval32(self, orc, golden, tables_npz, name):
        out = orc.dyadic_eval32(tables_npz[name].astype(np.float32), golden["lattice_u32"])
        assert np.array_equal(bits(out), bits(golden[f"{name}_eval32_out"]))

    @pytest.mark.parametrize("name", ["dyadic_linear_k15", "dyadic_cubic_k15"])
    def test_dyadic_eval64(self, orc, golden, tables_npz, name):
        out = orc.dyadic_eval(tables_npz[name], golden["u64"])
        assert np.array_equal(bits(out), bits(golden[f"{name}_eval_out"]))

    def test_dyadic_indices(self, orc, golden):
        assert np.array_equal(orc.dyadic_index(golden["u64"], 15), golden["dyadic_index_cap15"])
        v = np.minimum(golden["u64"], 1.0 - golden["u64"])
        assert np.array_equal(orc.dyadic_index(v, 1 << 62), golden["dyadic_index_uncapped"])
        assert np.array_equal(orc.dyadic_index(golden["pow2"], 64), golden["pow2_index"])
        assert np.array_equal(orc.dyadic_index32(golden["lattice_u32"], 15), golden["dyadic32_index_out"])
        assert np.array_equal(orc.dyadic_index32(golden["index32_probe"], 15), golden["index32_probe_out"])

    def test_ncchi2_eval(self, orc, golden, tables_npz):
        st, nu = tables_npz["ncchi2_cir_k64_stacks"], float(tables_npz["ncchi2_cir_k64_nu"])
        out = orc.ncchi2_eval(st, nu, golden["ncchi2_u"], golden["ncchi2_lam"])
        assert np.array_equal(bits(out), bits(golden["ncchi2_k64_perelem_out"]))
        out = orc.ncchi2_eval(st, nu, golden["ncchi2_u"], np.array([7.5]))
        assert np.array_equal(bits(out), bits(golden["ncchi2_k64_shared_out"]))

    def test_as241(self, orc, golden):
        u = golden["as241_u"]
        ref = golden["as241_out"]
        out = orc.as241_f64(u)
        central = np.abs(u - 0.5) <= 0.425
        # central branch: identical operation sequence, no transcendental -> bit-exact
        assert np.array_equal(bits(out[central]), bits(ref[central]))
        # tails depend on log (numpy SIMD vs libm, each <= 1 ulp): relative 1e-14
        np.testing.assert_allclose(out[~central], ref[~central], rtol=1e-14, atol=0)


class TestFusedAndFullSize:
    def test_fused_constant_matches_reference(self, orc, golden, tables_npz):
        n = 1 << 14
        out = orc.pcg32_constant_f32(42, 0, 0, tables_npz["constant_q10_l1"], n)
        assert np.array_equal(bits(out), bits(golden["const_q10_out"][:n].astype(np.float32)))

    def test_config1_full_hash(self, orc, hashes, tables_npz):
        out = orc.pcg32_constant_f32(42, 0, 0, tables_npz["constant_q10_l1"], 1 << 24)
        assert hashlib.sha256(out.tobytes()).hexdigest() == hashes["config1_const_q10_f32_sha256_2^24"]

    def test_dyadic_k15_full_hash(self, orc, hashes, tables_npz):
        out = orc.pcg32_dyadic_f32(42, 0, 0, tables_npz["dyadic_linear_k15"].astype(np.float32), 1 << 24)
        assert hashlib.sha256(out.tobytes()).hexdigest() == hashes["dyadic_linear_k15_f32_sha256_2^24"]


class TestSubDyadic:
    def test_degenerate_table_equals_reference_dyadic(self, orc, golden, tables_npz):
        """Sub-interval evaluator with K15 coefficients replicated over 8 slots
        must reproduce the reference dyadic_eval32 bit for bit (index + arithmetic)."""
        c = tables_npz["dyadic_linear_k15"].astype(np.float32)
        deg = np.repeat(c[:, 1:, None], 8, axis=2)
        out = orc.subdyadic_eval32(deg, 3, golden["lattice_u32"])
        assert np.array_equal(bits(out), bits(golden["dyadic_linear_k15_eval32_out"]))
        out = orc.pcg32_subdyadic_f32(42, 0, 0, deg, 3, 1 << 14)
        assert np.array_equal(bits(out), bits(golden["dyadic_linear_k15_eval32_out"][: 1 << 14]))

    def test_sub_interval_membership(self, orc, golden):
        """Label each slot with its own id: the selected slot's interval contains v."""
        K, b = 16, 3
        ids = np.arange(K * 8, dtype=np.float32).reshape(K, 8)
        c = np.stack([ids, np.zeros_like(ids)])  # z = id (c1 = 0)
        u = golden["lattice_u32"]
        z = orc.subdyadic_eval32(c, b, u)
        e = np.abs(z).astype(np.int64)
        j = e // 8 + 1
        s = e % 8
        v = np.minimum(u, np.float32(1) - u).astype(np.float64)
        a = 2.0 ** -(j + 1)
        lo = np.where(j < K, a + s * a / 8, 0.0)
        hi = np.where(j < K, a + (s + 1) * a / 8, 2.0**-K)
        assert np.all((lo <= v) & (v < hi))
        assert np.all(s[j == K] == 0)

    def test_shipped_table_error(self, orc, tables_npz):
        c = tables_npz["subdyadic_linear_k16_s8"].astype(np.float32)
        n = 1 << 20
        a = orc.pcg32_subdyadic_f32(42, 0, 0, c, 3, n)
        e = orc.pcg32_as241_f64(42, 0, 0, n)
        rmse = float(np.sqrt(np.mean((a - e) ** 2)))
        assert 2e-4 < rmse < 6e-4  # ~3.8e-4 (K15 reference layout: 6.4e-3)


class TestMlmcRestatement:
    def test_gbm_paths(self, orc, golden, hashes, tables_npz):
        lin = tables_npz["dyadic_linear_k15"]
        n = hashes["gbm_n_paths"]
        for scheme, payoff, level, n0 in hashes["gbm_cases"]:
            ref = golden[f"gbm_{scheme}_{payoff}_l{level}_n{n0}"]
            got = np.stack(orc.gbm_paths(mu=0.05, sigma=0.2, x0=1.0, t_end=1.0, level=level, n0=n0,
                                         milstein=scheme == "milstein", payoff_call=payoff == "call", strike=1.0,
                                         coeffs=lin, seed=42, seq=level << 32, n_paths=n))
            # approximate side: table + em_step only -> bit-exact
            assert np.array_equal(bits(got[2:]), bits(ref[2:])), (scheme, payoff, level, n0)
            # exact side goes through AS241 tails (log): relative 1e-13
            np.testing.assert_allclose(got[:2], ref[:2], rtol=1e-13, atol=1e-15)

    def test_cir_euler_paths(self, orc, golden, hashes, tables_npz):
        lin = tables_npz["dyadic_linear_k15"]
        for level, n0 in hashes["cir_euler_cases"]:
            ref = golden[f"cir_euler_l{level}_n{n0}"]
            got = np.stack(orc.cir_euler_paths(kappa=0.5, theta=0.04, sigma=0.2, x0=0.04, t_end=1.0, level=level,
                                               n0=n0, payoff_call=False, strike=1.0, coeffs=lin, seed=42,
                                               seq=(level << 32) | 5, n_paths=512))
            assert np.array_equal(bits(got[2:]), bits(ref[2:]))
            np.testing.assert_allclose(got[:2], ref[:2], rtol=1e-12, atol=1e-15)

    def test_cir_exact_paths(self, golden, hashes, tables_npz):
        from oracle import cir

        st, nu_t = tables_npz["ncchi2_cir_k16_stacks"], float(tables_npz["ncchi2_cir_k16_nu"])
        for level, n0 in hashes["cir_exact_cases"]:
            ref = golden[f"cir_exact_l{level}_n{n0}"]
            xe, xa, worst = cir.cir_exact_paths(kappa=0.5, theta=0.04, sigma=0.2, x0=0.04, t_end=1.0, level=level,
                                                n0=n0, stacks=st, nu_table=nu_t, seed=42, seq=level << 32,
                                                n_paths=256)
            assert np.array_equal(bits(xa), bits(ref[1]))
            np.testing.assert_allclose(xe, ref[0], rtol=1e-12)
            assert worst <= 1e-8

    @pytest.mark.parametrize("level,n0", [(0, 1), (1, 1), (3, 1), (2, 3)])
    def test_cir_milstein_restatement(self, orc, tables_npz, level, n0):
        """The oracle's truncated-Milstein CIR (no reference counterpart, SURVEY
        §8c "unpinned") against a numpy restatement built from the reference's
        own truncated-Euler loop (mlmc.py:289-331: uniforms, coupling, payoffs)
        with the Milstein term 1/2 b b'(dW^2 - dt) = sigma^2/4 (dW^2 - dt) of
        b(x) = sigma sqrt(x) added after the Euler step.  Same operation order,
        so both sides agree bit for bit; with the term removed it is the
        reference's scheme (pinned in test_cir_euler_paths)."""
        lin = tables_npz["dyadic_linear_k15"]
        kp, th, sg, x0 = 0.5, 0.04, 0.2, 0.04
        n, seq = 300, (level << 32) | 5
        got = np.stack(orc.cir_euler_paths(kappa=kp, theta=th, sigma=sg, x0=x0, t_end=1.0, level=level, n0=n0,
                                           payoff_call=False, strike=1.0, coeffs=lin, seed=42, seq=seq,
                                           n_paths=n, milstein=True))
        nf = n0 << level
        dt = 1.0 / nf
        sq = np.sqrt(dt)
        u = orc.u32_to_f64(orc.pcg32_words(42, seq, 0, nf * n)).reshape(nf, n)  # word k n_paths + p

        def step(x, dw, h):
            r = x + kp * (th - x) * h + sg * np.sqrt(np.abs(x)) * dw  # mlmc.py:295-296
            return r + 0.25 * sg * sg * (dw * dw - h)

        xs = {k: np.full(n, x0) for k in ("fe", "ce", "fa", "ca")}
        for pair in range(nf // 2):
            z1, z2 = orc.as241_f64(u[2 * pair]), orc.as241_f64(u[2 * pair + 1])
            w1, w2 = orc.dyadic_eval(lin, u[2 * pair]), orc.dyadic_eval(lin, u[2 * pair + 1])
            xs["fe"] = step(step(xs["fe"], sq * z1, dt), sq * z2, dt)
            xs["ce"] = step(xs["ce"], sq * (z1 + z2), 2.0 * dt)
            xs["fa"] = step(step(xs["fa"], sq * w1, dt), sq * w2, dt)
            xs["ca"] = step(xs["ca"], sq * (w1 + w2), 2.0 * dt)
        if nf % 2:
            xs["fe"] = step(xs["fe"], sq * orc.as241_f64(u[-1]), dt)
            xs["fa"] = step(xs["fa"], sq * orc.dyadic_eval(lin, u[-1]), dt)
        zero = np.zeros(n)
        want = np.stack([xs["fe"], xs["ce"] if level else zero, xs["fa"], xs["ca"] if level else zero])
        assert np.array_equal(bits(got), bits(want))
        # and it is not the Euler scheme
        eul = np.stack(orc.cir_euler_paths(kappa=kp, theta=th, sigma=sg, x0=x0, t_end=1.0, level=level, n0=n0,
                                           payoff_call=False, strike=1.0, coeffs=lin, seed=42, seq=seq,
                                           n_paths=n))
        assert not np.array_equal(eul[0], got[0])

"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle and
the reference's golden vectors.  Integer / index / f32 table work is
bit-exact; AS241 tails use a stated ulp-level tolerance."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    a = np.ascontiguousarray(a)
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


@pytest.fixture(scope="module")
def arv():
    import paper_2012_09715_b200 as arv

    return arv


def test_library_is_the_in_tree_build(arv):
    from paper_2012_09715_b200 import _native

    with open("/proc/self/maps") as fh:
        maps = fh.read()
    assert _native.LIB_PATH in maps


class TestPcg32Device:
    @pytest.mark.parametrize("offset,n", [(0, 4096), (3, 4093), (1 << 20, 100003), (2**40 + 5, 7)])
    def test_words(self, arv, orc, offset, n):
        s = arv.Pcg32Stream(42, 0, counter=offset)
        w = s.words(n)
        assert np.array_equal(w.cpu().numpy(), orc.pcg32_words(42, 0, offset, n))
        assert s.counter == offset + n

    def test_words_unaligned_output(self, arv, orc):
        buf = torch.empty(1001, dtype=torch.uint32, device="cuda")
        arv.Pcg32Stream(5, 9).words(1000, out=buf[1:])
        assert np.array_equal(buf[1:].cpu().numpy(), orc.pcg32_words(5, 9, 0, 1000))

    def test_uniform_f32(self, arv, orc):
        u = arv.Pcg32Stream(42, 0).uniforms(1 << 16)
        ref = orc.u32_to_f32(orc.pcg32_words(42, 0, 0, 1 << 16))
        assert np.array_equal(bits(u), bits(ref))

    def test_shards_concatenate(self, arv, orc):
        n = (1 << 18) + 3
        full = arv.Pcg32Stream(42, 0).sample(arv.load_table("subdyadic_linear_k16_s8"), n)
        parts = []
        for r in range(3):
            lo, hi = arv.shard_range(n, r, 3)
            parts.append(arv.Pcg32Stream(42, 0, counter=lo).sample(arv.load_table("subdyadic_linear_k16_s8"), hi - lo))
        assert np.array_equal(bits(torch.cat(parts)), bits(full))


class TestFusedGenerators:
    def test_constant_matches_reference(self, arv, golden):
        t = arv.load_table("constant_q10_l1")
        out = arv.Pcg32Stream(42, 0).sample(t, 1 << 14)
        assert np.array_equal(bits(out), bits(golden["const_q10_out"][: 1 << 14].astype(np.float32)))

    def test_config1_full_size_hash(self, arv, hashes):
        out = arv.Pcg32Stream(42, 0).sample(arv.load_table("constant_q10_l1"), 1 << 24)
        assert hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest() == hashes["config1_const_q10_f32_sha256_2^24"]

    def test_dyadic_k15_reference_layout(self, arv, golden, hashes):
        t = arv.load_table("dyadic_linear_k15")
        out = arv.Pcg32Stream(42, 0).sample(t, 1 << 14)
        assert np.array_equal(bits(out), bits(golden["dyadic_linear_k15_eval32_out"][: 1 << 14]))
        out = arv.Pcg32Stream(42, 0).sample(t, 1 << 24)
        assert hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest() == hashes["dyadic_linear_k15_f32_sha256_2^24"]

    def test_cubic_reference_layout(self, arv, orc, tables_npz):
        c = tables_npz["dyadic_cubic_k15"].astype(np.float32)
        out = arv.Pcg32Stream(3, 1).sample(arv.load_table("dyadic_cubic_k15"), 100001)
        assert np.array_equal(bits(out), bits(orc.pcg32_dyadic_f32(3, 1, 0, c, 100001)))

    @pytest.mark.parametrize("seed,sid,offset,n", [(42, 0, 0, 1 << 20), (1, 7, 12345, 99999), (42, 0, 1 << 27, 1 << 16)])
    def test_subdyadic_matches_oracle(self, arv, orc, tables_npz, seed, sid, offset, n):
        t = arv.load_table("subdyadic_linear_k16_s8")
        out = arv.Pcg32Stream(seed, sid, counter=offset).sample(t, n)
        ref = orc.pcg32_subdyadic_f32(seed, sid, offset, tables_npz["subdyadic_linear_k16_s8"].astype(np.float32), 3, n)
        assert np.array_equal(bits(out), bits(ref))

    def test_config2_full_size(self, arv, orc, tables_npz):
        """2^28 samples: chunk-wise bit-exact vs the oracle, and the error vs
        AS241-f64 of the same uniforms (size-independent property)."""
        n = 1 << 28
        t = arv.load_table("subdyadic_linear_k16_s8")
        out = arv.Pcg32Stream(42, 0).sample(t, n)
        c = tables_npz["subdyadic_linear_k16_s8"].astype(np.float32)
        for off in (0, n // 2, n - (1 << 20)):
            ref = orc.pcg32_subdyadic_f32(42, 0, off, c, 3, 1 << 20)
            assert np.array_equal(bits(out[off: off + (1 << 20)]), bits(ref))
        ex = arv.Pcg32Stream(42, 0).sample_exact64(n)
        err = out.double() - ex
        rmse = float(torch.sqrt(torch.mean(err * err)))
        assert 2e-4 < rmse < 6e-4
        assert bool(torch.isfinite(out).all())

    def test_antisymmetry_on_the_lattice(self, arv, orc, tables_npz):
        """test_sampler.py:137-139 / helpers.py:64-68: z(1 - u) == -z(u) bit for bit.
        The mirror of lattice word w is ~w (u -> 1 - u exactly), so the fused
        output of a stream is checked against the drop-in evaluator on 1 - u."""
        n = 1 << 20
        t = arv.load_table("subdyadic_linear_k16_s8")
        out = arv.Pcg32Stream(3, 8).sample(t, n).cpu().numpy()
        u = orc.u32_to_f32(orc.pcg32_words(3, 8, 0, n))
        mirrored = (np.float32(1.0) - u).astype(np.float32)
        assert np.array_equal(orc.u32_to_f32(~orc.pcg32_words(3, 8, 0, n)), mirrored)
        got = np.empty_like(mirrored)
        arv.get_kernels().subdyadic_eval32(tables_npz["subdyadic_linear_k16_s8"].astype(np.float32), 3, mirrored, got)
        assert np.array_equal(bits(got), bits(-out))

    @pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 15, 31, 33, 1023, 4097])
    @pytest.mark.parametrize("pad", [0, 1, 4])  # element offset into the buffer: v8 / scalar / v4 store paths
    def test_small_and_ragged(self, arv, orc, tables_npz, n, pad):
        sub = arv.load_table("subdyadic_linear_k16_s8")
        const = arv.load_table("constant_q10_l1")
        buf = torch.full((n + 16,), float("nan"), dtype=torch.float32, device="cuda")
        arv.Pcg32Stream(9, 4, counter=5).sample(sub, n, out=buf[pad:pad + n])
        ref = orc.pcg32_subdyadic_f32(9, 4, 5, tables_npz["subdyadic_linear_k16_s8"].astype(np.float32), 3, n)
        assert np.array_equal(bits(buf[pad:pad + n]), bits(ref))
        assert bool(torch.isnan(buf[pad + n:]).all()) and bool(torch.isnan(buf[:pad]).all())  # no overrun
        arv.Pcg32Stream(9, 4, counter=5).sample(const, n, out=buf[pad:pad + n])
        ref = orc.pcg32_constant_f32(9, 4, 5, tables_npz["constant_q10_l1"], n)
        assert np.array_equal(bits(buf[pad:pad + n]), bits(ref))

    def test_all_group_sizes_agree(self, arv):
        from paper_2012_09715_b200 import _native

        t = arv.load_table("subdyadic_linear_k16_s8")
        outs = []
        try:
            for group, ctas in ((8, 0), (8, 8), (4, 8), (8, 2), (4, 1), (4, 0)):
                _native.call("arv_set_tuning", 1, group)
                _native.call("arv_set_tuning", 2, ctas)
                outs.append(arv.Pcg32Stream(42, 0, counter=77).sample(t, 300001).cpu().numpy())
        finally:
            _native.call("arv_set_tuning", 1, 8)
            _native.call("arv_set_tuning", 2, 0)
        assert all(np.array_equal(bits(o), bits(outs[0])) for o in outs[1:])

    def test_unaligned_output(self, arv, orc, tables_npz):
        buf = torch.empty(10001, dtype=torch.float32, device="cuda")
        arv.Pcg32Stream(42, 0).sample(arv.load_table("subdyadic_linear_k16_s8"), 10000, out=buf[1:])
        ref = orc.pcg32_subdyadic_f32(42, 0, 0, tables_npz["subdyadic_linear_k16_s8"].astype(np.float32), 3, 10000)
        assert np.array_equal(bits(buf[1:]), bits(ref))

    def test_gaussian_f64_comparator(self, arv, orc):
        out = arv.Pcg32Stream(42, 0).sample_exact64(1 << 16).cpu().numpy()
        ref = orc.pcg32_as241_f64(42, 0, 0, 1 << 16)
        u = orc.u32_to_f32(orc.pcg32_words(42, 0, 0, 1 << 16)).astype(np.float64)
        central = np.abs(u - 0.5) <= 0.425
        assert np.array_equal(bits(out[central]), bits(ref[central]))
        np.testing.assert_allclose(out, ref, rtol=4e-16 * 8, atol=0)

    def test_gaussian_f32(self, arv, orc):
        out = arv.Pcg32Stream(42, 0).sample("exact", 1 << 16).cpu().numpy()
        ref = orc.pcg32_as241_f32(42, 0, 0, 1 << 16)
        ulp = np.abs(bits(out).astype(np.int64) - bits(ref).astype(np.int64))
        assert ulp.max() <= 4  # logf implementations differ by <= 1 ulp each
        ex = orc.pcg32_as241_f64(42, 0, 0, 1 << 16)
        np.testing.assert_allclose(out, ex, rtol=2e-6, atol=2e-6)


class TestDropInKernels:
    """The _kernels plugin functions on host (numpy) and device (torch) buffers."""

    def test_constant_eval(self, arv, golden, tables_npz):
        k = arv.get_kernels()
        v = tables_npz["constant_q10_l1"]
        u = golden["lattice_u32"].astype(np.float64)
        out = np.empty_like(u)
        k.constant_eval(v, u, out)
        assert np.array_equal(bits(out), bits(golden["const_q10_out"]))
        ud = torch.from_numpy(golden["u64"]).cuda()
        od = torch.empty_like(ud)
        k.constant_eval(v, ud, od)
        assert np.array_equal(bits(od), bits(golden["constant_u64_out"]))

    @pytest.mark.parametrize("name", ["dyadic_linear_k15", "dyadic_cubic_k15"])
    def test_dyadic_eval(self, arv, golden, tables_npz, name):
        k = arv.get_kernels()
        out = np.empty_like(golden["u64"])
        k.dyadic_eval(tables_npz[name], golden["u64"], out)
        assert np.array_equal(bits(out), bits(golden[f"{name}_eval_out"]))
        u32 = golden["lattice_u32"]
        o32 = np.empty_like(u32)
        k.dyadic_eval32(tables_npz[name].astype(np.float32), u32, o32)
        assert np.array_equal(bits(o32), bits(golden[f"{name}_eval32_out"]))

    def test_indices(self, arv, golden):
        k = arv.get_kernels()
        assert np.array_equal(k.dyadic_index(golden["u64"], 15), golden["dyadic_index_cap15"])
        v = np.minimum(golden["u64"], 1.0 - golden["u64"])
        assert np.array_equal(k.dyadic_index(v, 1 << 62), golden["dyadic_index_uncapped"])
        assert np.array_equal(k.dyadic_index(golden["pow2"], 64), golden["pow2_index"])
        assert np.array_equal(k.dyadic_index32(golden["lattice_u32"], 15), golden["dyadic32_index_out"])
        assert np.array_equal(k.dyadic_index32(golden["index32_probe"], 15), golden["index32_probe_out"])

    def test_ncchi2_eval(self, arv, golden, tables_npz):
        k = arv.get_kernels()
        st, nu = tables_npz["ncchi2_cir_k64_stacks"], float(tables_npz["ncchi2_cir_k64_nu"])
        out = np.empty_like(golden["ncchi2_u"])
        k.ncchi2_eval(st, nu, golden["ncchi2_u"], golden["ncchi2_lam"], out)
        assert np.array_equal(bits(out), bits(golden["ncchi2_k64_perelem_out"]))
        k.ncchi2_eval(st, nu, golden["ncchi2_u"], np.array([7.5]), out)
        assert np.array_equal(bits(out), bits(golden["ncchi2_k64_shared_out"]))

    def test_subdyadic_eval32(self, arv, orc, golden, tables_npz):
        k = arv.get_kernels()
        c = tables_npz["subdyadic_linear_k16_s8"].astype(np.float32)
        u = np.concatenate([golden["lattice_u32"], np.array([0.5, 0.25, 2.0**-20, 1e-30], np.float32)])
        out = np.empty_like(u)
        k.subdyadic_eval32(c, 3, u, out)
        assert np.array_equal(bits(out), bits(orc.subdyadic_eval32(c, 3, u)))

    def test_as241(self, arv, golden):
        u = golden["as241_u"]
        out = np.asarray(arv.gaussian_inv_cdf(u))
        ref = golden["as241_out"]
        central = np.abs(u - 0.5) <= 0.425
        assert np.array_equal(bits(out[central]), bits(ref[central]))
        np.testing.assert_allclose(out[~central], ref[~central], rtol=1e-14, atol=0)

    def test_sampler_wrappers(self, arv, golden, tables_npz):
        lin = arv.load_table("dyadic_linear_k15")
        assert arv.eval_dyadic(lin, 0.5) == 0.0
        assert arv.eval_dyadic(lin, 0.5, dtype=np.float32) == 0.0
        assert arv.dyadic_index(0.3) == 1 and arv.dyadic_index(2.0**-30, 15) == 15
        const = arv.load_table("constant_q10_l1")
        assert arv.eval_constant(const, 0.73) == const.values[747]
        assert arv.eval_constant(const, np.nextafter(1.0, 0.0)) == const.values[-1]
        with pytest.raises(arv.DomainError):
            arv.eval_ncchi2(arv.load_table("ncchi2_cir_k64_stacks"), 0.5, -1.0)
        with pytest.raises(arv.ConfigError):
            arv.eval_ncchi2(arv.load_table("ncchi2_cir_k64_stacks"), np.array([0.5, 0.6]), np.array([1.0, 2.0, 3.0]))
        with pytest.raises(arv.DomainError):
            arv.gaussian_inv_cdf(np.array([0.0, 0.5]))

    def test_fuzz_bit_patterns(self, arv, orc, tables_npz):
        """Random f64/f32 bit patterns in [0, 1] incl. subnormals, 0, 1/2 neighbours and
        exact powers of two: the drop-in kernels equal the oracle restatement (itself
        pinned to the reference) everywhere in the (0, 1) contract and never fault
        outside it (negative / > 1 / NaN inputs)."""
        k = arv.get_kernels()
        rng = np.random.default_rng(2024)
        raw = rng.integers(0, 0x3FF0000000000000, size=200_000, dtype=np.uint64)
        u = raw.view(np.float64).copy()
        u[:64] = [0.0, 1.0, 0.5, np.nextafter(0.5, 0), np.nextafter(0.5, 1), 5e-324, 2.0**-1022, 2.0**-1074] + \
            [2.0 ** -e for e in range(1, 57)]
        for name in ("dyadic_linear_k15", "dyadic_cubic_k15"):
            out = np.empty_like(u)
            k.dyadic_eval(tables_npz[name], u, out)
            inside = (u > 0) & (u < 1)
            assert np.array_equal(bits(out[inside]), bits(orc.dyadic_eval(tables_npz[name], u[inside])))
        assert np.array_equal(k.dyadic_index(u, 40), orc.dyadic_index(u, 40))
        u32 = raw.astype(np.uint32).view(np.float32)
        u32 = np.where((u32 >= 0) & (u32 <= 1), u32, np.float32(0.25)).astype(np.float32)
        out32 = np.empty_like(u32)
        k.dyadic_eval32(tables_npz["dyadic_linear_k15"].astype(np.float32), u32, out32)
        inside = (u32 > 0) & (u32 < 1)
        ref = orc.dyadic_eval32(tables_npz["dyadic_linear_k15"].astype(np.float32), u32[inside])
        assert np.array_equal(bits(out32[inside]), bits(ref))
        assert np.array_equal(k.dyadic_index32(u32, 15), orc.dyadic_index32(u32, 15))
        # out of contract: must not fault, values unspecified
        bad = np.array([-0.5, 1.5, np.nan, np.inf, -np.inf, -0.0, 2.0], dtype=np.float64)
        out = np.empty_like(bad)
        k.dyadic_eval(tables_npz["dyadic_linear_k15"], bad, out)
        k.constant_eval(tables_npz["constant_q10_l1"], bad, out)
        k.ncchi2_eval(tables_npz["ncchi2_cir_k64_stacks"], 2.0, bad, np.array([1.0]), out)
        torch.cuda.synchronize()

    @pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 1000, 4099, 70001])
    @pytest.mark.parametrize("pad_in,pad_out", [(0, 0), (1, 0), (0, 1), (2, 3)])
    def test_device_views_ragged(self, arv, orc, tables_npz, n, pad_in, pad_out):
        """Device-resident inputs at every alignment: 16-byte vector body plus
        scalar tail when the views are aligned, scalar grid-stride otherwise."""
        k = arv.get_kernels()
        rng = np.random.default_rng(n * 7 + pad_in)
        u = rng.random(n)
        lam = rng.random(n) * 300.0
        ud = torch.zeros(n + 8, dtype=torch.float64, device="cuda")
        ud[pad_in:pad_in + n] = torch.from_numpy(u).cuda()
        ld = torch.zeros(n + 8, dtype=torch.float64, device="cuda")
        ld[pad_in:pad_in + n] = torch.from_numpy(lam).cuda()
        uv, lv = ud[pad_in:pad_in + n], ld[pad_in:pad_in + n]
        o = torch.full((n + 8,), float("nan"), dtype=torch.float64, device="cuda")
        ov = o[pad_out:pad_out + n]

        def check(got, ref):
            assert np.array_equal(bits(got.cpu().numpy()), bits(np.asarray(ref)))
            assert torch.isnan(o[:pad_out]).all() and torch.isnan(o[pad_out + n:]).all()

        lin = tables_npz["dyadic_linear_k15"]
        k.dyadic_eval(lin, uv, ov)
        check(ov, orc.dyadic_eval(lin, u))
        cv = tables_npz["constant_q10_l1"]
        k.constant_eval(cv, uv, ov)
        check(ov, orc.constant_eval(cv, u))
        st, nu = tables_npz["ncchi2_cir_k64_stacks"], float(tables_npz["ncchi2_cir_k64_nu"])
        k.ncchi2_eval(st, nu, uv, lv, ov)
        check(ov, orc.ncchi2_eval(st, nu, u, lam))
        k.ncchi2_eval(st, nu, uv, torch.tensor([7.5], dtype=torch.float64, device="cuda"), ov)
        check(ov, orc.ncchi2_eval(st, nu, u, np.array([7.5])))
        k.gaussian_inv_cdf(uv, ov)  # tails go through log / sqrt: libm-level agreement
        got, ref = ov.cpu().numpy(), orc.as241_f64(u)
        central = np.abs(u - 0.5) <= 0.425
        assert np.array_equal(bits(got[central]), bits(ref[central]))
        np.testing.assert_allclose(got, ref, rtol=4e-16 * 8, atol=0)
        idx = k.dyadic_index(uv, 15)
        assert np.array_equal(idx.cpu().numpy(), orc.dyadic_index(u, 15))

        u32 = u.astype(np.float32)
        u32 = np.where(u32 >= 1.0, np.float32(0.5), u32)
        u32d = torch.zeros(n + 8, dtype=torch.float32, device="cuda")
        u32d[pad_in:pad_in + n] = torch.from_numpy(u32).cuda()
        u32v = u32d[pad_in:pad_in + n]
        o = torch.full((n + 8,), float("nan"), dtype=torch.float32, device="cuda")
        ov = o[pad_out:pad_out + n]
        k.dyadic_eval32(lin.astype(np.float32), u32v, ov)
        check(ov, orc.dyadic_eval32(lin.astype(np.float32), u32))
        c = tables_npz["subdyadic_linear_k16_s8"].astype(np.float32)
        k.subdyadic_eval32(c, 3, u32v, ov)
        check(ov, orc.subdyadic_eval32(c, 3, u32))
        k.gaussian_inv_cdf32(u32v, ov)
        got32 = ov.cpu().numpy()  # f32 rational after device vs glibc logf / sqrtf: a few ulp
        ulp = np.abs(bits(got32).astype(np.int64) - bits(orc.as241_f32(u32)).astype(np.int64))
        assert ulp.max() <= 8
        np.testing.assert_allclose(got32, orc.as241_f64(u32.astype(np.float64)), rtol=2e-6, atol=2e-6)
        assert np.array_equal(k.dyadic_index32(u32v, 15).cpu().numpy(), orc.dyadic_index32(u32, 15))

    def test_launch_counter_advances(self, arv):
        from paper_2012_09715_b200 import _native

        before = _native.launch_count()
        arv.Pcg32Stream(1, 1).sample(arv.load_table("constant_q10_l1"), 1000)
        assert _native.launch_count() == before + 1


def test_standalone_c_client(tmp_path, orc, tables_npz):
    """examples/c_abi_demo.c: a plain C program (no Python/torch) drives the C ABI."""
    import os
    import subprocess

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "c_abi_demo"
    subprocess.run(["gcc", "-O2", "-I", os.path.join(repo, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(repo, "examples", "c_abi_demo.c"),
                    "-L", os.path.join(repo, "paper_2012_09715_b200"), "-larv_b200", "-L", "/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{os.path.join(repo, 'paper_2012_09715_b200')}", "-o", str(exe)],
                   check=True)
    c = tables_npz["subdyadic_linear_k16_s8"].astype(np.float32)
    (tmp_path / "t.f32").write_bytes(c.tobytes())
    n = 1000003
    r = subprocess.run([str(exe), str(tmp_path / "t.f32"), str(n), str(tmp_path / "o.f32")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(tmp_path / "o.f32", dtype=np.float32)
    assert np.array_equal(bits(got), bits(orc.pcg32_subdyadic_f32(42, 0, 0, c, 3, n)))

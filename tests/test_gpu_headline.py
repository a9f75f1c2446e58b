"""GPU parity of the headline generator (config 2) beyond sampled chunks:

* the evaluators of the fused generators over the WHOLE f32 lattice (all 2^23
  values of w >> 9), for the shipped tables and random tables at every
  sub_bits the signed-table kernel takes, against the oracle;
* the signed-table kernel's exactness checks and its fallback (a table with
  an exact zero on the lattice, where the reference returns -0.0; a slope
  whose 2^-23 scaling is inexact);
* the full 2^28-sample config-2 output against the oracle's sha256;
* programmatic-dependent-launch ordering: a table written by the kernel that
  runs immediately before the generator on the stream is the one used.
"""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

LATTICE = 1 << 23


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.fixture(scope="module")
def arv():
    import paper_2012_09715_b200 as arv

    return arv


@pytest.fixture(scope="module")
def lattice_u():
    k = np.arange(LATTICE, dtype=np.float64)
    return ((k + 0.5) * 2.0**-23).astype(np.float32)


def lattice_eval(coeffs, sub_bits, mode):
    from paper_2012_09715_b200 import _device as dev
    from paper_2012_09715_b200._native import call

    c = torch.from_numpy(np.ascontiguousarray(coeffs, dtype=np.float32)).cuda()
    out = torch.empty(LATTICE, dtype=torch.float32, device="cuda")
    fast = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    call("arv_lattice_subdyadic_f32", c.data_ptr(), coeffs.shape[0] - 1, coeffs.shape[1], sub_bits, mode,
         out.data_ptr(), fast.data_ptr(), dev.stream_handle())
    return out.cpu().numpy(), int(fast.item())


def random_table(rng, K, b):
    """Degree-1 table shaped like a lower-tail ICDF fit: c1 > 0, z < 0 on (0, 1/2)."""
    c1 = rng.uniform(0.5, 40.0, size=(K, 1 << b))
    c0 = -(0.5 * c1) - rng.uniform(1e-3, 3.0, size=(K, 1 << b))
    return np.stack([c0, c1]).astype(np.float32)


@pytest.mark.parametrize("name,b", [("subdyadic_linear_k16_s8", 3), ("dyadic_linear_k15", 0)])
def test_shipped_tables_whole_lattice(arv, orc, tables_npz, lattice_u, name, b):
    if name == "dyadic_linear_k15":  # reference layout -> natural (2, K, 1): octave j -> ref[:, j]
        ref = tables_npz[name].astype(np.float32)
        c = np.ascontiguousarray(ref[:, 1:, None])
    else:
        c = tables_npz[name].astype(np.float32)
    want = orc.subdyadic_eval32(c, b, lattice_u)
    for mode in (0, 1, 2):
        got, fast = lattice_eval(c, b, mode)
        assert np.array_equal(bits(got), bits(want)), (name, mode)
        if mode:
            assert fast == 1, "shipped table must take the signed-table / lane-table fast path"


@pytest.mark.parametrize("b", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("K", [3, 16, 23, 30])
def test_random_tables_whole_lattice(arv, orc, lattice_u, b, K):
    rng = np.random.default_rng(100 * K + b)
    c = random_table(rng, K, b)
    want = orc.subdyadic_eval32(c, b, lattice_u)
    for mode in (1, 2):  # signed table, lane-private table (scalar and packed-pair forms)
        got, fast = lattice_eval(c, b, mode)
        assert fast == 1
        assert np.array_equal(bits(got), bits(want)), mode


def test_fallback_on_exact_zero(arv, orc, lattice_u):
    """A linear piece with an exact zero at a lattice point: the reference gives
    -0.0 on the upper half there, which the signed table cannot: the kernel
    must detect it and run the general evaluator."""
    rng = np.random.default_rng(7)
    c = random_table(rng, 16, 3)
    m = 3_500_001  # lattice point v = (m + 1/2) 2^-23 = 0.417 (octave 1)
    v = np.float32((m + 0.5) * 2.0**-23)
    c[1, 0, :] = 2.0
    c[0, 0, :] = -np.float32(2.0) * v  # exact
    want = orc.subdyadic_eval32(c, 3, lattice_u)
    zero = (want == 0) & (lattice_u < 0.5)
    assert zero.any() and np.signbit(orc.subdyadic_eval32(c, 3, (np.float32(1) - lattice_u[zero]))).all()
    for mode in (1, 2):
        got, fast = lattice_eval(c, 3, mode)
        assert fast == 0
        assert np.array_equal(bits(got), bits(want))
    # the fused generators take the same fallback: upper-half samples of that
    # point come out as -0.0 like the reference (signed-table kernel, then the
    # lane-table kernel that large calls take)
    n = 1 << 22
    want = bits(orc.pcg32_subdyadic_f32(11, 2, 0, c, 3, n))
    out = arv.Pcg32Stream(11, 2).sample(_subtable(arv, c, 3), n)
    assert np.array_equal(bits(out), want)
    with lane_min_n(20):
        out = arv.Pcg32Stream(11, 2).sample(_subtable(arv, c, 3), n)
    assert np.array_equal(bits(out), want)


def test_fallback_on_inexact_slope_scaling(arv, orc, lattice_u):
    rng = np.random.default_rng(8)
    c = random_table(rng, 12, 2)
    c[1, 4, 1] = np.float32(3e-36)  # c1 * 2^-23 is subnormal and would round
    for mode in (1, 2):  # (3e-36 2^-10 is subnormal too)
        got, fast = lattice_eval(c, 2, mode)
        assert fast == 0
        assert np.array_equal(bits(got), bits(orc.subdyadic_eval32(c, 2, lattice_u)))


import contextlib


@contextlib.contextmanager
def lane_min_n(log2n):
    """ARV_TUNE_LANE_MIN_N (key 5): calls of >= 2^log2n samples take the
    lane-table kernel (default 26); < 0 never."""
    from paper_2012_09715_b200._native import call

    call("arv_set_tuning", 5, log2n)
    try:
        yield
    finally:
        call("arv_set_tuning", 5, 26)


def _subtable(arv, c, b):
    from paper_2012_09715_b200.tables import SubDyadicTable

    return SubDyadicTable(degree=c.shape[0] - 1, n_octaves=c.shape[1], sub_bits=b, coeffs=c.astype(np.float64))


@pytest.mark.parametrize("b", [0, 1, 2, 4, 5])
def test_fused_generator_every_sub_bits(arv, orc, b):
    """The fused generator at each sub_bits (b <= 4 signed table, b = 5 general)."""
    rng = np.random.default_rng(b)
    c = random_table(rng, 18, b)
    n = (1 << 20) + 5
    want = bits(orc.pcg32_subdyadic_f32(42, 0, 3, c, b, n))
    out = arv.Pcg32Stream(42, 0, counter=3).sample(_subtable(arv, c, b), n)
    assert np.array_equal(bits(out), want)
    with lane_min_n(0):  # every call through the lane-table kernel (b <= 4; b = 5 stays general)
        out = arv.Pcg32Stream(42, 0, counter=3).sample(_subtable(arv, c, b), n)
    assert np.array_equal(bits(out), want)


@pytest.mark.parametrize("n", [1, 7, 8, 4097, (1 << 24) + 3])
def test_lane_kernel_ragged_sizes_and_alignment(arv, orc, n):
    """The lane-table kernel (512-thread CTAs, its own start-state walk) on
    ragged sizes, v8 / v4 store alignment and a non-zero stream offset."""
    tab = arv.load_table("subdyadic_linear_k16_s8")
    buf = torch.empty(n + 8, dtype=torch.float32, device="cuda")
    for shift in (0, 4):  # 32-byte (v8) and 16-byte (v4) aligned outputs
        out = buf[shift:shift + n]
        with lane_min_n(0):
            arv.Pcg32Stream(9, 4, counter=12345).sample(tab, n, out=out)
        m = min(n, 1 << 16)
        for lo in (0, n - m):
            want = orc.pcg32_subdyadic_f32(9, 4, 12345 + lo, tab.coeffs32, tab.sub_bits, m)
            assert np.array_equal(bits(out[lo:lo + m]), want.view(np.uint32)), (n, shift, lo)


def test_lane_kernel_threshold_is_bit_identical(arv):
    """Below / above ARV_TUNE_LANE_MIN_N the same call takes the signed-table
    or the lane-table kernel: identical output."""
    tab = arv.load_table("subdyadic_linear_k16_s8")
    n = (1 << 25) + 40
    with lane_min_n(-1):
        a = arv.Pcg32Stream(42, 0).sample(tab, n)
    with lane_min_n(0):
        b = arv.Pcg32Stream(42, 0).sample(tab, n)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_config2_full_output_sha256(arv, hashes):
    """All 2^28 config-2 samples, bit for bit (the oracle's full-output hash)."""
    out = arv.Pcg32Stream(42, 0).sample(arv.load_table("subdyadic_linear_k16_s8"), 1 << 28)
    h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()
    assert h == hashes["config2_subdyadic_f32_sha256_2^28"]


def test_pdl_table_written_by_previous_kernel(arv, orc, tables_npz):
    """The generator is launched with programmatic dependent launch; its table
    is staged after griddepcontrol.wait, so a table produced by the kernel
    just before it on the stream is the one used (no stale read)."""
    from paper_2012_09715_b200 import _device as dev
    from paper_2012_09715_b200._native import call

    base = tables_npz["subdyadic_linear_k16_s8"].astype(np.float32)
    src = torch.from_numpy(base).cuda()
    c = torch.zeros_like(src)
    n = 1 << 22
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    s = dev.stream_handle()
    for scale in (1.0, -1.0, 0.5, 2.0):
        # a long-running kernel, then the table-writing kernel, then the generator
        big = torch.empty(1 << 26, dtype=torch.float32, device="cuda")
        call("arv_store_probe", big.data_ptr(), big.numel(), s)
        ref = orc.pcg32_subdyadic_f32(42, 0, 0, (base * np.float32(scale)).astype(np.float32), 3, n)
        for lm in (26, 0):  # signed-table kernel, lane-table kernel
            c.zero_()
            call("arv_store_probe", big.data_ptr(), big.numel(), s)
            torch.mul(src, scale, out=c)
            with lane_min_n(lm):
                call("arv_pcg32_subdyadic_f32", 42, 0, 0, c.data_ptr(), 1, 16, 3, out.data_ptr(), n, s)
            assert np.array_equal(bits(out), bits(ref)), (scale, lm)


def test_config3_max_size_2_32_samples(arv, orc):
    """BASELINE config 3's largest single-GPU call: 2^32 samples (16 GiB) in one
    launch -- 64-bit group indices, > 2^31 outputs, the grid-stride tail --
    checked against the oracle at the start, across the 2^31 boundary and at
    the very end (sample i of the call = PCG32 output i)."""
    n = 1 << 32
    free, _ = torch.cuda.mem_get_info()
    if free < 4 * n + (2 << 30):
        pytest.skip("needs ~18 GiB of free device memory")
    tab = arv.load_table("subdyadic_linear_k16_s8")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    arv.Pcg32Stream(42, 0).sample(tab, n, out=out)
    m = 1 << 18
    for lo in (0, (1 << 31) - m // 2, n - m):
        want = orc.pcg32_subdyadic_f32(42, 0, lo, tab.coeffs32, tab.sub_bits, m)
        assert np.array_equal(bits(out[lo:lo + m]), want.view(np.uint32)), lo
    del out
    # a ragged size past 2^32 / 8 groups: the scalar tail of the last group
    n2 = (1 << 31) + 5
    out = torch.empty(n2, dtype=torch.float32, device="cuda")
    arv.Pcg32Stream(42, 0, counter=3).sample(tab, n2, out=out)
    want = orc.pcg32_subdyadic_f32(42, 0, 3 + n2 - m, tab.coeffs32, tab.sub_bits, m)
    assert np.array_equal(bits(out[n2 - m:]), want.view(np.uint32))


def test_sample_host_end_to_end_path(arv, orc):
    """Pcg32Stream.sample_host (the bench's e2e path): chunked generation with
    the D2H drained on a side stream into a pinned tensor or a numpy array --
    identical to the device samples, any chunking, the stream counter advanced;
    a buffer it could not fill in place is refused."""
    tab = arv.load_table("subdyadic_linear_k16_s8")
    n = (1 << 22) + 13
    dev_out = arv.Pcg32Stream(42, 5, counter=11).sample(tab, n)
    pinned = torch.empty(n, dtype=torch.float32, pin_memory=True)
    s = arv.Pcg32Stream(42, 5, counter=11)
    r = s.sample_host(tab, n, out=pinned, chunk=(1 << 20) + 4)
    assert r is pinned and s.counter == 11 + n
    assert np.array_equal(bits(pinned), bits(dev_out))
    host = np.empty(n, np.float32)
    arv.Pcg32Stream(42, 5, counter=11).sample_host(tab, n, out=host, chunk=1 << 21, sync=False)
    torch.cuda.synchronize()
    assert np.array_equal(host.view(np.uint32), bits(dev_out))
    auto = arv.Pcg32Stream(42, 5, counter=11).sample_host(tab, n)
    assert auto.is_pinned() and np.array_equal(bits(auto), bits(dev_out))
    with pytest.raises(arv.ConfigError):
        arv.Pcg32Stream(42, 5).sample_host(tab, 1000, out=np.empty(2000, np.float32)[::2])
    with pytest.raises(arv.ConfigError):
        arv.Pcg32Stream(42, 5).sample_host(tab, 1000, out=np.empty(999, np.float32))
    want = orc.pcg32_subdyadic_f32(42, 5, 11 + n - 4096, tab.coeffs32, tab.sub_bits, 4096)
    assert np.array_equal(host[-4096:].view(np.uint32), want.view(np.uint32))


def test_pdl_constant_table_written_by_previous_kernel(arv, orc, tables_npz):
    """The config-1 generator is launched with programmatic dependent launch
    too: its value table is staged after griddepcontrol.wait, so values written
    by the kernel just before it on the stream are the ones used, and
    back-to-back launches into one buffer keep their order."""
    from paper_2012_09715_b200 import _device as dev
    from paper_2012_09715_b200._native import call

    base = tables_npz["constant_q10_l1"].astype(np.float32)
    src = torch.from_numpy(base).cuda()
    v = torch.zeros_like(src)
    n = (1 << 22) + 24
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    big = torch.empty(1 << 26, dtype=torch.float32, device="cuda")
    s = dev.stream_handle()
    for scale in (1.0, -3.0, 0.25):
        v.zero_()
        call("arv_store_probe", big.data_ptr(), big.numel(), s)
        call("arv_pcg32_constant_f32", 1, 1, 0, src.data_ptr(), 10, out.data_ptr(), n, s)  # overwritten below
        torch.mul(src, scale, out=v)
        call("arv_pcg32_constant_f32", 42, 0, 7, v.data_ptr(), 10, out.data_ptr(), n, s)
        ref = orc.pcg32_constant_f32(42, 0, 7, (base * np.float32(scale)).astype(np.float32), n)
        assert np.array_equal(bits(out), bits(ref)), scale

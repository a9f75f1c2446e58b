"""The host-buffer (numpy) convention of the plugin: arv_host_* entry points
(csrc/arv_host.cu), which stage chunks through pinned buffers with the
copies and kernels overlapped.  Results must be bit-identical to the
device-buffer entry points and to the oracle for every length (chunk
boundaries, ragged tails, empty), every plugin function, shared and
per-element lambda, and for caller buffers the kernel cannot write directly
(strided, wrong dtype, 2-D)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def K():
    from paper_2012_09715_b200 import _kernels

    return _kernels


@pytest.fixture(scope="module")
def tabs(tables_npz):
    return {k: np.ascontiguousarray(v) for k, v in tables_npz.items()}


def u64(n, seed=1):
    rng = np.random.default_rng(seed)
    return rng.random(n) * (1 - 2**-40) + 2**-41


def same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


# lengths around the pipeline's chunking (>= 256 KiB chunks, 16 MiB slots,
# 3 slots) and tiny / empty calls
LENGTHS = [0, 1, 3, 4097, (1 << 15) + 1, (1 << 20) - 3, 3 * (1 << 21) + 7, (1 << 22) + 5]


@pytest.mark.parametrize("n", LENGTHS)
def test_dyadic_eval_host_equals_device_and_oracle(K, orc, tabs, n):
    u = u64(n, n)
    c = tabs["dyadic_linear_k15"]
    out = np.full(n, np.nan)
    K.dyadic_eval(c, u, out)
    assert same(out, orc.dyadic_eval(c, u))
    dev_out = torch.empty(n, dtype=torch.float64, device="cuda")
    K.dyadic_eval(c, torch.from_numpy(u).cuda(), dev_out)
    assert same(out, dev_out.cpu().numpy())


@pytest.mark.parametrize("n", LENGTHS)
def test_dyadic_eval32_host(K, orc, tabs, n):
    u = u64(n, 7 + n).astype(np.float32)
    c = tabs["dyadic_cubic_k15"].astype(np.float32)
    out = np.empty(n, np.float32)
    K.dyadic_eval32(c, u, out)
    assert same(out, orc.dyadic_eval32(c, u))


@pytest.mark.parametrize("n", [1, 5000, (1 << 21) + 3])
def test_index_and_constant_host(K, orc, tabs, n):
    u = u64(n, 3)
    assert same(K.dyadic_index(u, 15), orc.dyadic_index(u, 15))
    u32 = u.astype(np.float32)
    assert same(K.dyadic_index32(u32, 15), orc.dyadic_index32(u32, 15))
    out = np.empty(n)
    K.constant_eval(tabs["constant_q10_l1"], u, out)
    assert same(out, orc.constant_eval(tabs["constant_q10_l1"], u))


@pytest.mark.parametrize("n", [1, 4099, (1 << 21) + 11])
def test_ncchi2_host_shared_and_per_element_lambda(K, orc, tabs, n):
    st, nu = tabs["ncchi2_cir_k64_stacks"], float(np.asarray(tabs["ncchi2_cir_k64_nu"]).reshape(-1)[0])
    u = u64(n, 5)
    for lam in (np.array([7.5]), np.linspace(0.0, 400.0, n)):
        out = np.empty(n)
        K.ncchi2_eval(st, nu, u, lam, out)
        assert same(out, orc.ncchi2_eval(st, nu, u, lam))


def test_awkward_caller_buffers(K, orc, tabs):
    """Strided / wrong-dtype / 2-D buffers are written through a temporary and
    copied into the caller's array (never silently dropped)."""
    c = tabs["dyadic_linear_k15"]
    u = u64(10000, 9)
    want = orc.dyadic_eval(c, u)
    big = np.full(20000, np.nan)
    K.dyadic_eval(c, u, big[::2])  # strided view: written in place
    assert same(big[::2], want) and np.isnan(big[1::2]).all()
    o32 = np.empty(10000, np.float32)
    K.dyadic_eval(c, u, o32)  # wrong dtype: unsafe cast like np.copyto
    assert same(o32, want.astype(np.float32))
    o2 = np.empty((100, 100))
    K.dyadic_eval(c, u.reshape(100, 100), o2)
    assert same(o2.reshape(-1), want)
    ro = np.empty(10000)
    ro.setflags(write=False)
    with pytest.raises(ValueError):
        K.dyadic_eval(c, u, ro)


def test_sampler_layer_host_path(tabs, orc):
    """sampler.evaluate / eval_* on numpy inputs return numpy through the
    pipeline; scalars come back as Python numbers (sampler.py:97-206)."""
    import paper_2012_09715_b200 as arv

    lin = arv.load_table("dyadic_linear_k15")
    u = u64(3001, 2)
    got = arv.evaluate(lin, u)
    assert isinstance(got, np.ndarray) and same(got, orc.dyadic_eval(tabs["dyadic_linear_k15"], u))
    assert arv.eval_dyadic(lin, 0.5) == 0.0
    assert isinstance(arv.dyadic_index(0.3), int) and arv.dyadic_index(0.3) == 1
    out = np.empty(3001, np.float32)
    r = arv.eval_dyadic(lin, u, dtype=np.float32, out=out)
    assert r is out and same(out, orc.dyadic_eval32(tabs["dyadic_linear_k15"].astype(np.float32),
                                                   u.astype(np.float32)))
    z = arv.gaussian_inv_cdf(u)
    np.testing.assert_allclose(z, orc.as241_f64(u), rtol=1e-14)
    with pytest.raises(arv.DomainError):
        arv.gaussian_inv_cdf(np.array([0.5, 1.0]))


def test_host_pipeline_orders_with_the_callers_stream(K, orc, tabs):
    """The kernel runs on the caller's (torch current) stream: a table written
    by queued work on that stream is the one used."""
    c = torch.from_numpy(tabs["dyadic_linear_k15"]).cuda()
    src = c.clone()
    s = torch.cuda.Stream()
    u = u64(1 << 20, 4)
    with torch.cuda.stream(s):
        big = torch.empty(1 << 27, device="cuda")
        big.fill_(1.0)  # keep the stream busy
        c.mul_(2.0)
        out = np.empty(u.size)
        K.dyadic_eval(c, u, out)
    assert same(out, orc.dyadic_eval((src * 2.0).cpu().numpy(), u))


def test_host_pipeline_concurrent_callers(K, orc, tabs):
    """Python threads calling the plugin at once (ctypes releases the GIL): the
    per-device pipeline serialises them and every caller gets its own result."""
    from concurrent.futures import ThreadPoolExecutor

    c = tabs["dyadic_linear_k15"]
    us = [u64((1 << 21) + 17 * j, 100 + j) for j in range(6)]

    def work(u):
        out = np.empty_like(u)
        K.dyadic_eval(c, u, out)
        return out

    with ThreadPoolExecutor(6) as ex:
        outs = list(ex.map(work, us))
    for u, out in zip(us, outs):
        assert same(out, orc.dyadic_eval(c, u))

"""CUDA-graph capture of the C-ABI calls (verdict r1: remove the per-call host
cost of small requests).  Every generator / evaluator entry point only
enqueues work on the caller's stream (no host synchronisation, no allocation
inside the library), so a sequence of calls can be captured once with
torch.cuda.graph and replayed with one graph launch.  Kernel arguments
(PCG32 offsets included) are frozen at capture: a replay regenerates the
captured ranges."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def bits(t):
    return t.cpu().numpy().view(np.uint32)


def test_generator_calls_replay_from_a_graph(orc):
    import paper_2012_09715_b200 as arv

    sub = arv.load_table("subdyadic_linear_k16_s8")
    const = arv.load_table("constant_q10_l1")
    n, k = (1 << 20) + 8, 6
    out = torch.empty((k, n), dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up outside capture: tables uploaded, occupancy cached
        arv.Pcg32Stream(42, 0).sample(sub, n, out=out[0])
        arv.Pcg32Stream(42, 0).sample(const, n, out=out[1])
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    s = arv.Pcg32Stream(42, 0)
    with torch.cuda.graph(g):
        for i in range(k):
            s.sample(sub if i % 2 == 0 else const, n, out=out[i])
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    c = sub.coeffs32
    for i in range(k):
        if i % 2 == 0:
            want = orc.pcg32_subdyadic_f32(42, 0, i * n, c, sub.sub_bits, n)
        else:
            want = orc.pcg32_constant_f32(42, 0, i * n, const.values, n)
        assert np.array_equal(bits(out[i]), want.view(np.uint32)), i
    first = out.clone()
    g.replay()  # frozen offsets: the same samples again
    torch.cuda.synchronize()
    assert torch.equal(first, out)


def test_lane_table_kernel_replays_from_a_graph(orc):
    """A call through the lane-table headline kernel (59 KB of opted-in dynamic
    shared memory, set per call) captures and replays as well."""
    import paper_2012_09715_b200 as arv
    from paper_2012_09715_b200._native import call

    call("arv_set_tuning", 5, 24)  # ARV_TUNE_LANE_MIN_N: lane-table kernel from 2^24 samples (default 2^26)

    sub = arv.load_table("subdyadic_linear_k16_s8")
    n = (1 << 24) + 16
    out = torch.empty((2, n), dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        arv.Pcg32Stream(42, 0).sample(sub, n, out=out[0])
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    s = arv.Pcg32Stream(42, 3)
    with torch.cuda.graph(g):
        for i in range(2):
            s.sample(sub, n, out=out[i])
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    m = 1 << 16
    for i in range(2):
        for lo in (0, n - m):
            want = orc.pcg32_subdyadic_f32(42, 3, i * n + lo, sub.coeffs32, sub.sub_bits, m)
            assert np.array_equal(bits(out[i, lo:lo + m]), want.view(np.uint32)), (i, lo)
    call("arv_set_tuning", 5, 26)


def test_dropin_eval_replays_from_a_graph(orc, tables_npz):
    from paper_2012_09715_b200 import _kernels

    c = torch.from_numpy(tables_npz["dyadic_linear_k15"]).cuda()
    u = torch.rand(1 << 18, dtype=torch.float64, device="cuda") * (1 - 2**-40) + 2**-41
    out = torch.empty_like(u)
    _kernels.dyadic_eval(c, u, out)  # warm-up
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        _kernels.dyadic_eval(c, u, out)
    u.copy_(torch.rand_like(u) * (1 - 2**-40) + 2**-41)  # new inputs in the captured buffer
    g.replay()
    torch.cuda.synchronize()
    want = orc.dyadic_eval(tables_npz["dyadic_linear_k15"], u.cpu().numpy())
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want.view(np.uint64))

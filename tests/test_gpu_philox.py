"""GPU replay of the reference's own uniform stream (Philox-4x64-10).

With ``PhiloxStream`` / ``level_stream(..., generator="philox")`` the device
reproduces the reference's UniformStream bit for bit, so evaluate() and the
MLMC pilots are compared against the REAL reference outputs (tests/golden,
made by approxrv itself, no stream substitution)."""

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


def test_words_and_uniforms(arv, golden, orc):
    s = arv.PhiloxStream(42, 7)
    assert np.array_equal(s.raw_words(64).cpu().numpy(), golden["philox_words_42_7"])
    assert s.counter == 64
    u = arv.PhiloxStream(5, (3 << 32) | 1, counter=13).uniforms(4099)
    assert np.array_equal(bits(u), bits(golden["philox_uniforms_5_3_c13"]))
    big = arv.PhiloxStream(1, 2, counter=(1 << 40) + 3).uniforms(1 << 20)
    assert np.array_equal(bits(big), bits(orc.philox_uniforms(1, 2, (1 << 40) + 3, 1 << 20)))


def test_fused_evaluate_matches_reference(arv, golden):
    lin = arv.load_table("dyadic_linear_k15")
    const = arv.load_table("constant_q10_l1")
    assert np.array_equal(bits(arv.PhiloxStream(42, 9).sample(lin, 8192)), bits(golden["philox_eval_dyadic_lin"]))
    assert np.array_equal(bits(arv.PhiloxStream(42, 9).sample(const, 8192)), bits(golden["philox_eval_const"]))
    ex = arv.PhiloxStream(42, 9).sample("exact", 8192).cpu().numpy()
    ref = golden["philox_eval_exact"]
    u = arv.PhiloxStream(42, 9).uniforms(8192).cpu().numpy()
    central = np.abs(u - 0.5) <= 0.425
    assert np.array_equal(bits(ex[central]), bits(ref[central]))
    np.testing.assert_allclose(ex, ref, rtol=1e-14, atol=0)


def test_sample_coupled_matches_reference(arv, golden):
    """sampler.sample_coupled (sampler.py:209-218) on the reference's own stream."""
    lin = arv.load_table("dyadic_linear_k15")
    b = arv.sample_coupled(arv.PhiloxStream(42, 9), lin, 8192)
    assert np.array_equal(bits(b.z_approx), bits(golden["philox_eval_dyadic_lin"]))
    np.testing.assert_allclose(b.z_exact.cpu().numpy(), golden["philox_eval_exact"], rtol=1e-14, atol=0)
    assert len(b) == 8192


def test_gbm_replays_reference_paths(arv, golden, hashes):
    lin = arv.load_table("dyadic_linear_k15")
    gbm = arv.GbmParams(0.05, 0.2, 1.0, 1.0)
    for scheme, payoff, level, n0 in hashes["philox_gbm_cases"]:
        spec = arv.LevelSpec(level=level, scheme=scheme, process=gbm, rv_source=lin, kind="four_way",
                             payoff=payoff, strike=1.0, n0=n0)
        b = arv.simulate(spec, arv.level_stream(42, level, generator="philox"), 1000)
        got = torch.stack([b.p_fine_exact, b.p_coarse_exact, b.p_fine_approx, b.p_coarse_approx]).cpu().numpy()
        ref = golden[f"philox_gbm_{scheme}_{payoff}_l{level}_n{n0}"]
        assert np.array_equal(bits(got[2:]), bits(ref[2:])), (scheme, payoff, level, n0)
        np.testing.assert_allclose(got[:2], ref[:2], rtol=1e-13, atol=1e-15)
        # the reference's estimate_level_suite on the same paths
        suite = arv.estimate_level_suite(spec, arv.level_stream(42, level, generator="philox"), 1000)
        rs = golden[f"philox_suite_{scheme}_{payoff}_l{level}_n{n0}"]
        for row, key in enumerate(("two_way_exact", "two_way_approx", "four_way")):
            np.testing.assert_allclose(suite[key].mean, rs[row, 0], rtol=1e-11, atol=1e-16)
            np.testing.assert_allclose(suite[key].variance, rs[row, 1], rtol=1e-9, atol=1e-20)


def test_aligned_vector_path(arv, orc):
    """4-word-aligned counters take the 16-byte-store path; ragged tails and
    mid-block starts the scalar one -- both bit-exact with the oracle."""
    for counter, n in ((0, (1 << 16) + 3), (4, 4097), (8, 1), (12, 6)):
        u = arv.PhiloxStream(9, 4, counter=counter).uniforms(n)
        assert np.array_equal(bits(u), bits(orc.philox_uniforms(9, 4, counter, n))), (counter, n)
        w = arv.PhiloxStream(9, 4, counter=counter).raw_words(n).cpu().numpy()
        assert np.array_equal(w, orc.philox_words(9, 4, counter, n)), (counter, n)

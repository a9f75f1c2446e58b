"""CPU emulation of the level kernels' per-tile warp reduction (csrc/arv_mlmc.cu,
warp_sum5): the transposed reduction of five values per lane must build, for
every value, exactly the summation tree of the plain xor-butterfly
(`s += shfl_xor(s, o)` for o = 16, 8, 4, 2, 1), so that the (count, mean, M2)
statistics are bit-identical to the per-value butterflies it replaced."""

import numpy as np


def butterfly(x):
    """x: (32,) doubles of one value; returns what every lane holds after the butterfly."""
    s = x.copy()
    for o in (16, 8, 4, 2, 1):
        s = s + s[np.arange(32) ^ o]
    return s


def warp_sum5(x):
    """x: (5, 32).  Returns (c, e) as in the kernel: c holds value 0 / 1 / 2 / 3 in lanes
    [0, 8) / [16, 24) / [8, 16) / [24, 32), e value 4 in every lane."""
    lane = np.arange(32)
    h16, h8 = (lane & 16) != 0, (lane & 8) != 0
    keep_a, send_a = np.where(h16, x[1], x[0]), np.where(h16, x[0], x[1])
    keep_b, send_b = np.where(h16, x[3], x[2]), np.where(h16, x[2], x[3])
    a = keep_a + send_a[lane ^ 16]
    b = keep_b + send_b[lane ^ 16]
    c = np.where(h8, b, a) + np.where(h8, a, b)[lane ^ 8]
    e = x[4] + x[4][lane ^ 16]
    e = e + e[lane ^ 8]
    for o in (4, 2, 1):
        c = c + c[lane ^ o]
        e = e + e[lane ^ o]
    return c, e


def test_transposed_reduction_builds_the_butterfly_tree():
    rng = np.random.default_rng(3)
    for scale in (1.0, 1e-8, 1e12):
        for _ in range(200):
            x = rng.standard_normal((5, 32)) * scale * rng.uniform(0.1, 10.0, size=(5, 1))
            x[:, rng.integers(0, 32, size=5)] = 0.0  # invalid lanes contribute +0.0
            c, e = warp_sum5(x)
            want = [butterfly(x[k]) for k in range(5)]
            for k, lanes in ((0, range(0, 8)), (1, range(16, 24)), (2, range(8, 16)), (3, range(24, 32))):
                for ln in lanes:
                    assert c[ln].tobytes() == want[k][0].tobytes(), (k, ln)
            assert all(e[ln].tobytes() == want[4][0].tobytes() for ln in range(32))
            # the butterfly itself leaves the same value in every lane (so lane 0 is "the" result)
            assert all(np.all(w.view(np.uint64) == w.view(np.uint64)[0]) for w in want)

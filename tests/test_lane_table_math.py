"""CPU check of the lane-table index construction of the headline kernel
(csrc/arv_sample.cu, EvalLinLane), over the whole f32 lattice.

With i = (int32)w >> 9 the kernel builds vh = (i + 1/2) 2^-13 exactly in f32
(magic 0x44C00000 + i, minus 1536, plus 2^-14), truncates it to f16 and uses
the top 6 + b bits of the f16 pattern (sign | E5 | sub-interval) as the table
row.  The reference's index is the octave of v = min(u, 1 - u)
(_kernels.pyx:26-53: 126 - (bits >> 23)) and, for the sub-interval tables,
the top b mantissa bits of v.  This test restates both in numpy and checks
that they agree at every lattice point, that the f32 construction is exact,
and that the rows stay inside the 55 KB table.
"""

import numpy as np
import pytest


@pytest.mark.parametrize("b", [0, 3, 4])
def test_lane_table_rows_match_reference_index(b):
    k = np.arange(1 << 23, dtype=np.int64)              # lattice index: u = (k + 1/2) 2^-23
    w = (k << 9).astype(np.uint32)
    i = (w.view(np.int32) >> 9).astype(np.int64)        # k, or k - 2^23 for u >= 1/2
    # the kernel's f32 arithmetic, step by step (every result must be exact)
    g = (np.uint32(0x44C00000) + i.astype(np.uint32)).view(np.float32)
    assert np.array_equal(g.astype(np.float64), (12582912 + i) * 2.0**-13)
    vh = (g - np.float32(1536.0)) + np.float32(2.0**-14)
    assert vh.dtype == np.float32
    assert np.array_equal(vh.astype(np.float64), (i + 0.5) * 2.0**-13)
    # f16 truncation (cvt.rz) of a value in the normal f16 range, on the bit pattern
    bits = vh.view(np.uint32).astype(np.int64)
    e8 = (bits >> 23) & 0xFF
    assert e8.min() >= 113 and e8.max() <= 135           # |vh| in [2^-14, 2^9): E5 = 1 .. 23
    h = ((bits >> 31) << 15) | ((e8 - 112) << 10) | ((bits & 0x7FFFFF) >> 13)
    row = h >> (10 - b)
    # the reference index: v = min(u, 1 - u) on the lattice, octave and sub-interval
    u = ((k + 0.5) * 2.0**-23).astype(np.float32)
    v = np.where(u < 0.5, u, np.float32(1.0) - u).astype(np.float32)
    vb = v.view(np.uint32).astype(np.int64)
    octave = 126 - (vb >> 23)                             # 1 .. 23
    sub = (vb & 0x7FFFFF) >> (23 - b) if b else np.zeros_like(vb)
    sign = (u >= 0.5).astype(np.int64)
    want = (sign << (5 + b)) | ((24 - octave) << b) | sub
    assert np.array_equal(row, want)
    # rows E5 = 0 (the 2^b rows below the table, 1 KB) are never addressed; the last row ends at 56 KB
    row_bytes = 1 << (10 - b)
    assert (row * row_bytes).min() >= 1024 and ((row + 1) * row_bytes).max() <= 56 * 1024
    # and |vh| = v 2^10: the slope stored in the table is c1 2^-10
    assert np.array_equal(np.abs(vh).astype(np.float64), v.astype(np.float64) * 1024.0)

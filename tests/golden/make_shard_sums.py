"""Per-rank checksums of the config-2 bench output (bench.py --gpus N).

Rank r of the bench generates outputs [r 2^28, (r+1) 2^28) of PCG32(42, 0)
through the 16x8 sub-interval table.  The checksum is the sum of the shard's
64-bit words modulo 2^64 (an order-independent device reduction).  Made with
the oracle (TEST INFRASTRUCTURE) for r = 0..7 into tests/golden/hashes.json.
"""

import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    c = np.load(os.path.join(HERE, "..", "..", "paper_2012_09715_b200", "data", "tables.npz"))[
        "subdyadic_linear_k16_s8"].astype(np.float32)
    n, ch = 1 << 28, 1 << 24

    def part(off):
        a = oracle.pcg32_subdyadic_f32(42, 0, off, c, 3, ch)
        return int(a.view(np.uint64).sum(dtype=np.uint64))

    sums = []
    with ThreadPoolExecutor(os.cpu_count() or 8) as ex:
        for r in range(8):
            s = sum(ex.map(part, range(r * n, (r + 1) * n, ch))) % (1 << 64)
            sums.append(str(s))
    p = os.path.join(HERE, "hashes.json")
    with open(p) as fh:
        h = json.load(fh)
    h["config2_shard_word_sums_mod2^64"] = sums
    with open(p, "w") as fh:
        json.dump(h, fh, indent=1)
    print(sums)


if __name__ == "__main__":
    main()

"""Multi-rank host logic on CPU: world_size 2 over gloo (127.0.0.1).

The data path has no collective: sample shards are PCG32 offset ranges and
MLMC path shards are contiguous path ranges.  The only exchange is the merge
of per-level (count, mean, M2) triples (mlmc.allreduce_triples), exercised
here with gloo exactly as bench.py / estimate_level_suite run it over NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle
        from paper_2012_09715_b200.mlmc import NSLOT, allreduce_triples
        from paper_2012_09715_b200.sampler import shard_range

        # --- MLMC: per-rank path shard -> triples -> merged stats ----------------
        rng = np.random.default_rng(7)
        full = rng.normal(0.0, 1.0, size=(NSLOT, 100_003)) * np.arange(1, NSLOT + 1)[:, None] + 1.05
        lo, hi = shard_range(full.shape[1], rank, WORLD)
        mine = full[:, lo:hi]
        tri = np.stack([np.full(NSLOT, mine.shape[1], dtype=np.float64), mine.mean(1),
                        ((mine - mine.mean(1, keepdims=True)) ** 2).sum(1)], axis=1)
        merged = allreduce_triples(torch.from_numpy(tri)).numpy()

        # --- sampling: each rank's PCG32 offset shard of the fused generator -------
        lin = np.load(os.path.join(os.path.dirname(oracle.__file__), "..", "paper_2012_09715_b200", "data",
                                   "tables.npz"))["subdyadic_linear_k16_s8"].astype(np.float32)
        n = (1 << 16) + 12
        slo, shi = shard_range(n, rank, WORLD)
        part = oracle.pcg32_subdyadic_f32(42, 0, slo, lin, 3, shi - slo)
        parts = [None] * WORLD
        dist.all_gather_object(parts, (slo, shi, part))
        q.put((rank, merged, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_merge_and_shards(tables_npz, orc):
    from paper_2012_09715_b200.mlmc import NSLOT

    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    full = rng.normal(0.0, 1.0, size=(NSLOT, 100_003)) * np.arange(1, NSLOT + 1)[:, None] + 1.05
    for rank, merged, parts in results:
        assert np.all(merged[:, 0] == full.shape[1])
        np.testing.assert_allclose(merged[:, 1], full.mean(1), rtol=1e-13)
        np.testing.assert_allclose(merged[:, 2] / (full.shape[1] - 1), full.var(1, ddof=1), rtol=1e-11)
        # shards tile the stream and concatenate to the single-process output bit for bit
        parts = sorted(parts, key=lambda t: t[0])
        assert parts[0][0] == 0 and parts[0][1] == parts[1][0]
        cat = np.concatenate([p[2] for p in parts])
        ref = orc.pcg32_subdyadic_f32(42, 0, 0, tables_npz["subdyadic_linear_k16_s8"].astype(np.float32), 3,
                                      cat.size)
        assert np.array_equal(cat.view(np.uint32), ref.view(np.uint32))
    # both ranks agree exactly
    assert np.array_equal(results[0][1], results[1][1])

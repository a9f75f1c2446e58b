"""Two ranks (torch.distributed.run, gloo, sharing the GPU): the sharded MLMC
pilot -- contiguous path ranges per rank, per-kind (count, mean, M2) merged by
two all-reduces -- equals the single-process pilot over the same paths."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
def test_sharded_pilot_equals_single_process(tmp_path):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "dist_worker.py"),
           str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=540)
    assert r.returncode == 0, r.stderr[-3000:]
    ranks = [json.load(open(tmp_path / f"rank{i}.json")) for i in range(2)]
    assert ranks[0] == ranks[1]  # both ranks hold the merged statistics
    for key, (n, mean, var, fn, fmean, fvar) in ranks[0].items():
        assert n == fn == 30011, key
        assert mean == pytest.approx(fmean, rel=1e-12, abs=1e-18), key
        assert var == pytest.approx(fvar, rel=1e-10, abs=1e-22), key

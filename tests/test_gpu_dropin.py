"""The drop-in, checked from the reference's side of the plugin boundary.

``tests/golden/make_golden_r2.py`` ran the reference's own sampler / mlmc /
metrics code (``sampler.evaluate``, ``eval_dyadic``, ``eval_ncchi2``,
``sample_coupled``, ``mlmc.estimate_level_suite``, ``mlmc.simulate`` for GBM,
CIR-exact and CIR-Euler, ``metrics.rmse_ncchi2``) with its plugin slot
(``sampler.kernels``, _backend.py:14-24) wrapped in a recorder around the
compiled reference kernels, and stored every plugin call: the arguments exactly
as the reference passes them (numpy dtypes and shapes, scalar batches, shared
and per-element lambda, caller-allocated ``out``) and what the call wrote or
returned.  Replaying every call through ``paper_2012_09715_b200._kernels`` with
the same numpy arguments and getting the same bits back means the reference's
code, whose work between plugin calls is deterministic numpy, computes the
same results with the CUDA plugin swapped in.
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def trace():
    with open(os.path.join(GOLDEN, "dropin_trace.json")) as fh:
        manifest = json.load(fh)
    with np.load(os.path.join(GOLDEN, "dropin_trace.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    return manifest, arrays


def _label_of(labels, i):
    cur = "?"
    for start, lab in labels:
        if start <= i:
            cur = lab
    return cur


def _replay(kernels, manifest, arrays, make_out):
    n_checked = 0
    for i, call in enumerate(manifest["calls"]):
        args, outs = [], {}
        for j, a in enumerate(call["args"]):
            if "scalar" in a:
                args.append(a["scalar"])
                continue
            src = arrays[f"c{i}_a{j}"]
            if a["out"]:
                buf = make_out(src)
                outs[j] = buf
                args.append(buf)
            else:
                args.append(src.copy())
        ret = getattr(kernels, call["name"])(*args)
        where = f"call {i} {call['name']} ({_label_of(manifest['labels'], i)})"
        for j, buf in outs.items():
            got = buf.cpu().numpy() if isinstance(buf, torch.Tensor) else buf
            want = arrays[f"c{i}_o{j}"]
            assert got.dtype == want.dtype and got.shape == want.shape, where
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), where
            n_checked += 1
        if call.get("ret"):
            want = arrays[f"c{i}_ret"]
            got = ret.cpu().numpy() if isinstance(ret, torch.Tensor) else np.asarray(ret)
            assert got.dtype == want.dtype, where
            assert np.array_equal(got, want), where
            n_checked += 1
    return n_checked


def test_reference_call_trace_replays_bit_exact(trace):
    """Every plugin call of the reference's own code, host (numpy) buffers."""
    from paper_2012_09715_b200 import _kernels

    manifest, arrays = trace
    n = _replay(_kernels, manifest, arrays, make_out=lambda src: np.full_like(src, np.nan))
    assert n == len(manifest["calls"])


def test_reference_call_trace_replays_with_device_out(trace):
    """Same calls, caller's ``out`` a CUDA tensor (the zero-copy convention)."""
    from paper_2012_09715_b200 import _kernels

    manifest, arrays = trace
    n = _replay(_kernels, manifest, arrays,
                make_out=lambda src: torch.full(src.shape, float("nan"),
                                                dtype=getattr(torch, str(src.dtype)), device="cuda"))
    assert n == len(manifest["calls"])


def test_trace_covers_every_plugin_function(trace):
    manifest, _ = trace
    names = {c["name"] for c in manifest["calls"]}
    # the reference's own callers never reach dyadic_index32: sampler.dyadic_index
    # coerces every batch to f64 first (sampler.py:91-94,111-124); it is pinned
    # against the compiled reference directly in test_gpu_parity.py
    assert names == {"constant_eval", "dyadic_index", "dyadic_eval", "dyadic_eval32", "ncchi2_eval"}
    # the MLMC estimators are in the trace, and their summary is the reference's
    assert any("estimate_level_suite" in lab for _, lab in manifest["labels"])


def test_backend_selects_cuda_plugin():
    """_backend.py mirror: the plugin module is ours and reports COMPILED."""
    from paper_2012_09715_b200 import _backend, _kernels

    assert _backend.kernels is _kernels
    assert _kernels.COMPILED is True

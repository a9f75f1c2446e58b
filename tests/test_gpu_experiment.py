"""End-to-end MLMC experiment driver vs the reference's run_experiment
(cli.py:248-329) on the same config, replaying the reference's Philox streams."""

import csv
import json
import os

import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "experiment_ref")


def read_levels(path):
    out = {}
    with open(path) as fh:
        for row in csv.DictReader(fh):
            out[(int(row["level"]), row["source"], row["estimator"], row["statistic"])] = float(row["value"])
    return out


def test_experiment_matches_reference(tmp_path):
    from paper_2012_09715_b200 import experiment

    cfg = json.load(open(os.path.join(REF, "config.json")))
    cfg["generator"] = "philox"
    summary = experiment.run_experiment(cfg, tmp_path)
    ours = read_levels(tmp_path / "levels.csv")
    ref = read_levels(os.path.join(REF, "levels.csv"))
    assert set(ours) == set(ref)
    for key, v in ref.items():
        if key[3] == "cost_per_path_seconds":
            continue  # wall clock (CPU vs B200)
        assert ours[key] == pytest.approx(v, rel=2e-9, abs=1e-20), key
    with open(os.path.join(REF, "allocation.csv")) as fh:
        ref_alloc = list(csv.reader(fh))
    with open(tmp_path / "allocation.csv") as fh:
        our_alloc = list(csv.reader(fh))
    for r, o in zip(ref_alloc[1:], our_alloc[1:]):
        assert r[0] == o[0] and r[1] == o[1] and r[3] == o[3]  # same path counts per level
        assert float(o[2]) == pytest.approx(float(r[2]), rel=1e-9)
    assert "linear:15" in summary["sources"]


def test_nested_estimate_runs():
    import paper_2012_09715_b200 as arv
    from paper_2012_09715_b200 import experiment

    gbm = arv.GbmParams(0.05, 0.2, 1.0, 1.0)
    lin = arv.load_table("dyadic_linear_k15")
    res = experiment.nested_estimate("euler_maruyama", gbm, lin, [0, 1, 2, 3], [400000, 100000, 50000, 25000],
                                     [2000, 1000, 500, 250], seed=7)
    # E[X_T] under EM with 2^3 * 2 steps is (1 + 0.05/16)^16 ~ exp(0.05)
    assert abs(res["estimate"] - (1 + 0.05 / 16) ** 16) < 5 * res["std_error"] + 1e-4


def test_device_rmse_grid_matches_reference(golden):
    """metrics.rmse_ncchi2 (metrics.py:324-350) regenerated on the device."""
    import numpy as np

    import paper_2012_09715_b200 as arv
    from paper_2012_09715_b200 import metrics

    tabs = [arv.load_table("ncchi2_nu1_k16_stacks"), arv.load_table("ncchi2_cir_k16_stacks")]
    grid = metrics.rmse_ncchi2(tabs, golden["rmse_grid_lambdas"], n_samples=1 << 14)
    assert not grid.failures
    # exact quantiles agree to the |F - u| <= 1e-9 tolerance of both Newton solvers
    np.testing.assert_allclose(grid.values, golden["rmse_grid_values"], rtol=1e-6)
    # published Table 5a, nu = 1 column (reproduce.py:30-37)
    np.testing.assert_allclose(grid.values[:, 0], [0.036, 0.045, 0.054, 0.098, 0.134, 0.186], atol=0.0025)

"""End-to-end MLMC experiment driver on the device (mirrors approxrv/cli.py:195-329).

``run_experiment(cfg, out_dir)`` takes the reference's flat ``key = value``
experiment configuration (process, scheme, seed, pilot, epsilon, n0, payoff,
strike, levels, sources, process parameters), runs every level's pilot as one
fused device kernel (``mlmc.estimate_level_suite`` / ``estimate_level``),
computes the regular and nested optimal allocations, and writes the same
``levels.csv``, ``allocation.csv`` and ``experiment.json`` as the reference.

Extensions:
  * ``generator = philox`` replays the reference's own UniformStream, so the
    pilot statistics match the reference run path for path; the default is
    ``pcg32``.
  * ``nested_estimate`` runs the nested estimator itself with the allocated
    path counts (cheap two-way terms + four-way corrections) and returns the
    telescoped mean and its standard error.

Table sources are the shipped tables or ARVT files (table fitting is an
offline reference step): exact | constant:10 | linear:15 | cubic:15 |
ncchi2:1:15 (ncchi2 with the process nu) | file:<path>.

    python -m paper_2012_09715_b200.experiment --config exp.cfg --out-dir results
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import sys
from pathlib import Path

from . import mlmc
from .errors import ConfigError
from .tableio import import_table
from .tables import load_table, shipped_names


def parse_experiment_config(path) -> dict:
    """Flat ``key = value`` file; '#' starts a comment (cli.py:195-210)."""
    cfg = {}
    try:
        text = Path(path).read_text()
    except OSError as exc:
        raise ConfigError(f"cannot read config file {path}: {exc}") from exc
    for ln, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"{path}:{ln}: expected 'key = value', got {raw!r}")
        key, _, val = line.partition("=")
        cfg[key.strip().lower()] = val.strip()
    return cfg


def parse_levels(text: str) -> list[int]:
    text = text.strip()
    if ":" in text:
        lo, hi = text.split(":")
        return list(range(int(lo), int(hi) + 1))
    return [int(x) for x in text.replace(",", " ").split()]


def source_from_spec(text: str, nu: float | None):
    """(table or "exact", label) for a source spec (cli.py:213-237 syntax)."""
    text = text.strip()
    if text == "exact":
        return "exact", text
    head, _, rest = text.partition(":")
    if head == "file":
        return import_table(rest), text
    if head == "constant" and rest == "10":
        return load_table("constant_q10_l1"), text
    if head in ("linear", "cubic") and rest == "15":
        return load_table(f"dyadic_{head}_k15"), text
    if head == "dyadic" and rest in ("1:15", "3:15"):
        return load_table("dyadic_linear_k15" if rest == "1:15" else "dyadic_cubic_k15"), text
    if head == "ncchi2":
        if nu is None:
            raise ConfigError("ncchi2 sources need a CIR process (nu comes from it)")
        if rest == "1:15":
            for name in ("ncchi2_cir_k16_stacks", "ncchi2_nu1_k16_stacks", "ncchi2_cir_k64_stacks"):
                t = load_table(name)
                if t.nu == nu:
                    return t, text
    raise ConfigError(f"source {text!r} is not shipped ({shipped_names()}); fit it with approxrv and pass file:<path>")


def _process(cfg: dict):
    kind = cfg.get("process", "gbm").lower()
    if kind == "gbm":
        return mlmc.GbmParams(mu=float(cfg.get("mu", 0.05)), sigma=float(cfg.get("sigma", 0.2)),
                              x0=float(cfg.get("x0", 1.0)), t_end=float(cfg.get("t_end", 1.0))), None, kind
    if kind == "cir":
        p = mlmc.CirParams(kappa=float(cfg.get("kappa", 0.5)), theta=float(cfg.get("theta", 1.0)),
                           sigma=float(cfg.get("sigma", 1.0)), x0=float(cfg.get("x0", 1.0)),
                           t_end=float(cfg.get("t_end", 1.0)))
        return p, 4.0 * p.kappa * p.theta / p.sigma**2, kind
    raise ConfigError(f"unknown process {kind!r}")


def _write_rows(path: Path, header, rows) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)


def run_experiment(cfg: dict, out_dir) -> dict:
    """Pilot every level on the device, allocate, write the reference's outputs."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    process, nu, kind = _process(cfg)
    scheme = cfg.get("scheme", "euler_maruyama").lower()
    seed = int(cfg.get("seed", 0))
    pilot = int(cfg.get("pilot", 20000))
    epsilon = float(cfg.get("epsilon", 0.01))
    n0 = int(cfg.get("n0", 2 if kind == "gbm" else 4))
    payoff = cfg.get("payoff", "identity")
    strike = float(cfg.get("strike", 1.0))
    levels = parse_levels(cfg.get("levels", "0:4"))
    generator = cfg.get("generator", "pcg32").lower()
    sources = [s.strip() for s in cfg.get("sources", "exact").split(",") if s.strip()]

    rows, alloc_rows = [], []
    summary = {"config": dict(cfg), "sources": {}, "device": "cuda-sm100a"}
    for text in sources:
        source, label = source_from_spec(text, nu)
        per_level = {}
        for lvl in levels:
            stream = mlmc.level_stream(seed, lvl, generator=generator)
            if source == "exact":
                spec = mlmc.LevelSpec(level=lvl, scheme=scheme, process=process, rv_source="exact",
                                      kind="two_way", payoff=payoff, strike=strike, n0=n0)
                stats = {"two_way_exact": mlmc.estimate_level(spec, stream, pilot)}
            else:
                spec = mlmc.LevelSpec(level=lvl, scheme=scheme, process=process, rv_source=source,
                                      kind="four_way", payoff=payoff, strike=strike, n0=n0)
                stats = mlmc.estimate_level_suite(spec, stream, pilot)
            per_level[lvl] = stats
            for key, st in stats.items():
                for stat_name, value in (("mean", st.mean), ("variance", st.variance),
                                         ("cost_per_path_seconds", st.cost_per_path_seconds),
                                         ("cost_per_path_draws", st.cost_per_path_draws),
                                         ("n_paths", st.n_paths)):
                    rows.append([lvl, label, key, stat_name, f"{value:.10e}"])
        if source == "exact" or scheme != "cir_exact":
            key = "two_way_exact" if source == "exact" else "two_way_approx"
            alloc = mlmc.optimal_allocation([per_level[lv][key] for lv in levels], epsilon)
            alloc_rows.append([label, "regular", f"{alloc.predicted_cost:.6e}",
                               " ".join(str(x) for x in alloc.n_paths)])
            entry = {"regular_cost": alloc.predicted_cost, "paths": alloc.n_paths}
            if source != "exact":
                cheap, corr, total = mlmc.optimal_allocation_nested(
                    [per_level[lv]["two_way_approx"] for lv in levels],
                    [per_level[lv]["four_way"] for lv in levels], epsilon)
                alloc_rows.append([label, "nested", f"{total:.6e}",
                                   " ".join(f"{a}/{b}" for a, b in zip(cheap.n_paths, corr.n_paths))])
                entry["nested_cost"] = total
                entry["nested_paths"] = {"cheap": cheap.n_paths, "correction": corr.n_paths}
        else:
            entry = {"correction_log2_gap": {
                lv: math.log2(per_level[lv]["correction"].variance / per_level[lv]["plain_exact"].variance)
                for lv in levels if per_level[lv]["plain_exact"].variance > 0
                and per_level[lv]["correction"].variance > 0}}
        summary["sources"][label] = entry

    _write_rows(out_dir / "levels.csv", ["level", "source", "estimator", "statistic", "value"], rows)
    _write_rows(out_dir / "allocation.csv", ["source", "estimator", "predicted_cost", "paths_per_level"], alloc_rows)
    with open(out_dir / "experiment.json", "w") as fh:
        json.dump(summary, fh, indent=2, default=float)
    return summary


def nested_estimate(scheme: str, process, source, levels, cheap_paths, corr_paths, *, seed: int = 0,
                    n0: int = 2, payoff: str = "identity", strike: float = 1.0, generator: str = "pcg32") -> dict:
    """Run the nested MLMC estimator: sum over levels of the cheap two-way mean
    (table side, ``cheap_paths[l]`` paths, batch 1) plus the exact-minus-
    approximate four-way correction (``corr_paths[l]`` paths, batch 2), on
    streams disjoint from the pilots (level_stream batch index 1 / 2)."""
    total, var = 0.0, 0.0
    per = []
    for lvl, m, mm in zip(levels, cheap_paths, corr_paths):
        spec = mlmc.LevelSpec(level=lvl, scheme=scheme, process=process, rv_source=source, kind="four_way",
                              payoff=payoff, strike=strike, n0=n0)
        cheap = mlmc.estimate_level_suite(spec, mlmc.level_stream(seed, lvl, 1, generator=generator), max(m, 100))
        corr = mlmc.estimate_level_suite(spec, mlmc.level_stream(seed, lvl, 2, generator=generator), max(mm, 100))
        c, f = cheap["two_way_approx"], corr["four_way"]
        total += c.mean + f.mean
        var += c.variance / c.n_paths + f.variance / f.n_paths
        per.append({"level": lvl, "cheap_mean": c.mean, "correction_mean": f.mean,
                    "cheap_paths": c.n_paths, "correction_paths": f.n_paths})
    return {"estimate": total, "std_error": math.sqrt(var), "levels": per}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="approxrv-b200-mlmc")
    ap.add_argument("--config", required=True)
    ap.add_argument("--out-dir", default="mlmc_results")
    args = ap.parse_args(argv)
    try:
        run_experiment(parse_experiment_config(args.config), args.out_dir)
    except ConfigError as exc:  # cli.py:406-414 exit-code contract
        print(f"error: {exc}", file=sys.stderr)
        return 2
    print(f"wrote {args.out_dir}/levels.csv, allocation.csv, experiment.json")
    return 0


if __name__ == "__main__":
    sys.exit(main())

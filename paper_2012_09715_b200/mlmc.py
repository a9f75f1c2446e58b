"""Nested multilevel Monte Carlo on the device (mirrors approxrv/mlmc.py).

Parameter and spec types keep the reference's names, fields and validation
(mlmc.py:38-120).  A level's coupled simulation (fine/coarse x exact/approx
from the same uniforms) runs as ONE fused kernel with one thread per path
(csrc/arv_mlmc.cu); only the per-kind (count, mean, M2) triples come back.

Streams: ``level_stream(seed, level, batch)`` is the PCG32 stream
``(seed, (level << 32) | batch)`` (mlmc.py:414-416); the uniform of fine
step k on path p is output ``k * n_paths + p`` -- the reference's addressing
with Philox words replaced by PCG32 outputs.  Paths therefore shard across
GPUs by contiguous ranges with bit-identical per-path results, and the only
exchange is a merge of the per-kind triples (``estimate_level_suite`` with a
``torch.distributed`` group: two all-reduces of 15 doubles).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Union

import numpy as np
import torch

from . import _device as dev
from . import _native as nat
from .errors import ConfigError, NumericalError
from .sampler import PhiloxStream, Pcg32Stream
from .tables import ConstantTable, DyadicPolyTable, NcChi2Table, SubDyadicTable, load_table

SIDES = ("exact", "approx", "both")
SCHEMES = ("euler_maruyama", "milstein", "cir_exact", "cir_euler_truncated", "cir_milstein_truncated")
KINDS = ("plain", "two_way", "four_way")
PAYOFFS = ("identity", "call")
_SCHEME_CODE = {
    "euler_maruyama": nat.SCHEME_EM,
    "milstein": nat.SCHEME_MILSTEIN,
    "cir_exact": nat.SCHEME_CIR_EXACT,
    "cir_euler_truncated": nat.SCHEME_CIR_EULER_TRUNCATED,
    "cir_milstein_truncated": nat.SCHEME_CIR_MILSTEIN_TRUNCATED,
}
# Slot order of the kernels' statistics (include/approxrv_b200.h ARV_NKIND).
SLOTS = ("two_way_exact", "two_way_approx", "four_way", "plain_exact", "plain_approx")
NSLOT = len(SLOTS)


@dataclass(frozen=True)
class GbmParams:
    """Geometric Brownian motion dX = mu X dt + sigma X dW (mlmc.py:38-49)."""

    mu: float
    sigma: float
    x0: float
    t_end: float

    def __post_init__(self):
        if not (self.sigma > 0 and self.x0 > 0 and self.t_end > 0):
            raise ConfigError("GBM requires sigma > 0, x0 > 0, t_end > 0")


@dataclass(frozen=True)
class CirParams:
    """CIR process dX = kappa (theta - X) dt + sigma sqrt(X) dW (mlmc.py:52-69)."""

    kappa: float
    theta: float
    sigma: float
    x0: float
    t_end: float

    def __post_init__(self):
        for name in ("kappa", "theta", "sigma", "x0", "t_end"):
            if not getattr(self, name) > 0:
                raise ConfigError(f"CIR requires {name} > 0")

    @property
    def feller_satisfied(self) -> bool:
        return 2.0 * self.kappa * self.theta >= self.sigma**2

    @property
    def nu(self) -> float:
        return 4.0 * self.kappa * self.theta / (self.sigma * self.sigma)


@dataclass(frozen=True)
class LevelSpec:
    """One MLMC level (mlmc.py:72-120); validation identical to the reference."""

    level: int
    scheme: str
    process: Union[GbmParams, CirParams]
    rv_source: Union[str, ConstantTable, DyadicPolyTable, NcChi2Table] = "exact"
    kind: str = "two_way"
    payoff: str = "identity"
    strike: float = 1.0
    n0: int = 2

    def __post_init__(self):
        if self.level < 0:
            raise ConfigError("level must be >= 0")
        if self.scheme not in SCHEMES:
            raise ConfigError(f"unknown scheme {self.scheme!r}")
        if self.kind not in KINDS:
            raise ConfigError(f"unknown kind {self.kind!r}")
        if self.payoff not in PAYOFFS:
            raise ConfigError(f"unknown payoff {self.payoff!r}")
        if self.n0 < 1:
            raise ConfigError("n0 must be >= 1")
        if self.kind == "four_way" and _is_exact(self.rv_source):
            raise ConfigError("four-way differences need a table source")
        gaussian = self.scheme in ("euler_maruyama", "milstein", "cir_euler_truncated", "cir_milstein_truncated")
        if isinstance(self.process, GbmParams) and self.scheme.startswith("cir"):
            raise ConfigError("CIR schemes need CirParams")
        if isinstance(self.process, CirParams) and not self.scheme.startswith("cir"):
            raise ConfigError(f"scheme {self.scheme!r} needs GbmParams")
        if not _is_exact(self.rv_source):
            if gaussian and _is_ncchi2(self.rv_source):
                raise ConfigError("Gaussian schemes need a Gaussian table source")
            if self.scheme == "cir_exact" and not _is_ncchi2(self.rv_source):
                raise ConfigError("cir_exact needs an NcChi2Table source")

    @property
    def n_steps_fine(self) -> int:
        return self.n0 << self.level

    @property
    def dt_fine(self) -> float:
        return self.process.t_end / self.n_steps_fine


def _is_exact(src) -> bool:
    return isinstance(src, str) and src == "exact"


def _is_ncchi2(src) -> bool:
    return isinstance(src, NcChi2Table) or type(src).__name__ == "NcChi2Table"


@dataclass
class LevelStats:
    """Sample statistics of one level's difference estimator (mlmc.py:138-149)."""

    level: int
    kind: str
    mean: float
    variance: float
    n_paths: int
    cost_per_path_seconds: float
    cost_per_path_draws: float
    degenerate: bool = False


@dataclass(frozen=True)
class PathBatch:
    """Per-path terminal payoffs (device tensors), mlmc.py:123-135."""

    p_fine_exact: Optional[torch.Tensor]
    p_coarse_exact: Optional[torch.Tensor]
    p_fine_approx: Optional[torch.Tensor]
    p_coarse_approx: Optional[torch.Tensor]
    draws_per_path: int


def level_stream(seed: int, level: int, batch_index: int = 0, generator: str = "pcg32"):
    """Deterministic disjoint stream for (level, batch) workers (mlmc.py:414-416).

    ``generator="philox"`` gives the reference's own UniformStream words
    (Philox-4x64-10), so device paths replay the reference path by path;
    the default is PCG32 (BASELINE.json).
    """
    sid = (level << 32) | batch_index
    if generator == "philox":
        return PhiloxStream(seed, stream_id=sid)
    if generator != "pcg32":
        raise ConfigError(f"unknown generator {generator!r}")
    return Pcg32Stream(seed, stream_id=sid)


# ---------------------------------------------------------------------------
# Kernel driver
# ---------------------------------------------------------------------------

_DEFAULT_GAUSS = "dyadic_linear_k15"


def _gauss_coeffs(src) -> np.ndarray:
    if _is_exact(src):
        # the kernel takes a table argument; with sides="exact" (the only sides
        # an exact source allows) the approximate side is never evaluated
        src = load_table(_DEFAULT_GAUSS)
    if isinstance(src, ConstantTable) or type(src).__name__ == "ConstantTable":
        # (1, 2^q): "degree 0" = piecewise constant, evaluated as constant_eval
        v = np.asarray(src.values, dtype=np.float64).reshape(1, -1)
        v.setflags(write=False)
        return _cached_row(src, v)
    if isinstance(src, SubDyadicTable):
        raise ConfigError("the device path kernels take reference-layout Gaussian tables")
    if getattr(src, "decay", 0.5) != 0.5:
        raise ConfigError("the device path kernels require decay rate 1/2")
    return src.coeffs


_ROWS: dict = {}


def _cached_row(table, arr):
    hit = _ROWS.get(id(table))
    if hit is None or hit[0] is not table:
        hit = _ROWS[id(table)] = (table, arr)
    return hit[1]


def _ncchi2_table(spec: LevelSpec):
    if not _is_exact(spec.rv_source):
        return spec.rv_source
    nu = spec.process.nu
    for name in ("ncchi2_cir_k64_stacks", "ncchi2_cir_k16_stacks", "ncchi2_nu1_k16_stacks"):
        t = load_table(name)
        if t.nu == nu:
            return t  # used only as the Newton warm start
    raise ConfigError("cir_exact with rv_source='exact' needs a table of matching nu for the warm start")


_SIDES_CODE = {"both": nat.SIDES_BOTH, "exact": nat.SIDES_EXACT, "approx": nat.SIDES_APPROX}


def _native_spec(spec: LevelSpec, stream: Pcg32Stream, n_paths: int, path_lo: int, path_count: int,
                 sides: str = "both"):
    p = spec.process
    s = nat.LevelSpec()
    if isinstance(p, GbmParams):
        s.a, s.b, s.c = p.mu, p.sigma, 0.0
    else:
        s.a, s.b, s.c = p.kappa, p.theta, p.sigma
    s.x0, s.t_end = p.x0, p.t_end
    s.level, s.n0 = spec.level, spec.n0
    s.scheme = _SCHEME_CODE[spec.scheme]
    s.payoff = nat.PAYOFF_CALL if spec.payoff == "call" else nat.PAYOFF_IDENTITY
    s.strike = spec.strike
    s.seed, s.stream_id = int(stream.seed), int(stream.stream_id)
    s.n_paths_total, s.path_lo, s.path_count = n_paths, path_lo, path_count
    s.rng = nat.RNG_PHILOX if isinstance(stream, PhiloxStream) else nat.RNG_PCG32
    s.sides = _SIDES_CODE[sides]
    return s


def _workspace_bytes(spec: LevelSpec, count: int, device) -> int:
    ws_bytes = int(nat.lib.arv_mlmc_workspace_bytes(count))
    if spec.scheme == "cir_exact":
        # segmented CIR levels (records re-bucketed by lambda between segments,
        # ~84 B per path) up to an eighth of the device memory; else the
        # one-kernel form
        # (device properties are cached; cudaMemGetInfo costs ~0.1 ms per call)
        seg_bytes = int(nat.lib.arv_mlmc_cir_workspace_bytes(count))
        if seg_bytes <= torch.cuda.get_device_properties(device).total_memory // 8:
            ws_bytes = seg_bytes
    return ws_bytes


def run_level(spec: LevelSpec, stream: Pcg32Stream, n_paths: int, *, path_lo: int = 0,
              path_count: Optional[int] = None, want_paths: bool = False, device=None, sides: str = "both",
              stats_out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
              n_fail_out: Optional[torch.Tensor] = None):
    """Launch one level; returns (stats device f64[NSLOT,3], paths or None, n_fail or None).

    The stream's counter is not consulted: paths are addressed from output
    0 of (seed, stream_id) as in the reference's fresh ``level_stream``.
    ``sides`` ("both", "exact", "approx") skips the other side's work; its
    payoffs and statistics slots are then unspecified.  ``stats_out``
    (f64[NSLOT * 3]), ``workspace`` (uint8, at least the level's workspace
    bytes) and ``n_fail_out`` (int64[1], accumulated into) let a caller that
    launches many levels on one stream reuse its buffers (stream order keeps
    the reuse safe).
    """
    device = device or dev.require_cuda()
    count = n_paths - path_lo if path_count is None else path_count
    if n_paths < 1 or count < 1:
        raise ConfigError("need at least one path")
    ns = _native_spec(spec, stream, n_paths, path_lo, count, sides)
    stats = stats_out if stats_out is not None else torch.empty(NSLOT * 3, dtype=torch.float64, device=device)
    paths = torch.empty((4, count), dtype=torch.float64, device=device) if want_paths else None
    ws_bytes = _workspace_bytes(spec, count, device)
    if workspace is not None and workspace.numel() >= ws_bytes:
        ws = workspace
    else:
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    s = dev.stream_handle(device)
    pp = paths.data_ptr() if paths is not None else None
    n_fail = None
    if spec.scheme == "cir_exact":
        tab = _ncchi2_table(spec)
        st = dev.table_on_device(tab.eval_stacks, torch.float64, device)
        n_fail = n_fail_out if n_fail_out is not None else torch.zeros(1, dtype=torch.int64, device=device)
        nat.call("arv_mlmc_cir_exact_level", nat.C.byref(ns), st.data_ptr(), st.shape[1], st.shape[2] - 1,
                 st.shape[3], float(tab.nu), stats.data_ptr(), pp, n_fail.data_ptr(), ws.data_ptr(), ws_bytes, s)
    else:
        c = dev.table_on_device(_gauss_coeffs(spec.rv_source), torch.float64, device)
        nat.call("arv_mlmc_gaussian_level", nat.C.byref(ns), c.data_ptr(), c.shape[0] - 1, c.shape[1],
                 stats.data_ptr(), pp, ws.data_ptr(), ws_bytes, s)
    return stats.view(NSLOT, 3), paths, n_fail


def _sides_for(spec: LevelSpec) -> str:
    """mlmc.py:156-161: both sides for four-way levels, else the source's side."""
    if spec.kind == "four_way":
        return "both"
    return "exact" if _is_exact(spec.rv_source) else "approx"


def _resolve_sides(spec: LevelSpec, sides: Optional[str]) -> str:
    sides = sides or _sides_for(spec)
    if sides not in SIDES:
        raise ConfigError(f"unknown sides {sides!r}")
    if sides in ("approx", "both") and _is_exact(spec.rv_source):
        raise ConfigError("approximate side requested but rv_source is 'exact'")  # mlmc.py:181-182
    return sides


def simulate(spec: LevelSpec, stream: Pcg32Stream, n_paths: int, sides: Optional[str] = None) -> PathBatch:
    """Coupled fine/coarse x exact/approx payoffs per path (mlmc.py:334-338).

    ``sides`` as in the reference (mlmc.py:176-192, 221-229): the payoffs of
    an unrequested side are ``None`` and the kernel does not compute them.
    """
    sides = _resolve_sides(spec, sides)
    _, paths, n_fail = run_level(spec, stream, n_paths, want_paths=True, sides=sides)
    _check_fail(spec, n_fail)
    ex, ap = sides in ("exact", "both"), sides in ("approx", "both")
    return PathBatch(paths[0] if ex else None, paths[1] if ex else None, paths[2] if ap else None,
                     paths[3] if ap else None, draws_per_path=spec.n_steps_fine)


def simulate_gbm_coupled(spec: LevelSpec, stream, n_paths: int, sides: Optional[str] = None) -> PathBatch:
    """mlmc.py:164-229: GBM Euler-Maruyama / Milstein coupled paths."""
    if spec.scheme not in ("euler_maruyama", "milstein"):
        raise ConfigError(f"simulate_gbm_coupled cannot run scheme {spec.scheme!r}")
    return simulate(spec, stream, n_paths, sides)


def simulate_cir_coupled(spec: LevelSpec, stream, n_paths: int, sides: Optional[str] = None) -> PathBatch:
    """mlmc.py:232-331: CIR exact / truncated Euler (and truncated Milstein) coupled paths."""
    if spec.scheme in ("euler_maruyama", "milstein"):
        raise ConfigError(f"simulate_cir_coupled cannot run scheme {spec.scheme!r}")
    return simulate(spec, stream, n_paths, sides)


def difference(spec_kind: str, rv_source, batch: PathBatch):
    """The per-path difference a level estimates (mlmc.py:341-353), on the device."""
    if spec_kind == "plain":
        return batch.p_fine_exact if _is_exact(rv_source) else batch.p_fine_approx
    if spec_kind == "two_way":
        if _is_exact(rv_source):
            return batch.p_fine_exact - batch.p_coarse_exact
        return batch.p_fine_approx - batch.p_coarse_approx
    if spec_kind != "four_way":
        raise ConfigError(f"unknown level kind {spec_kind!r}")
    return batch.p_fine_exact - batch.p_coarse_exact - batch.p_fine_approx + batch.p_coarse_approx


def telescoped_mean(specs: list, seed: int, n_pilot: int, generator: str = "pcg32") -> tuple:
    """Sum of per-level means with its combined standard error (mlmc.py:553-561)."""
    total, var_sum = 0.0, 0.0
    for spec in specs:
        stats = estimate_level(spec, level_stream(seed, spec.level, generator=generator), n_pilot)
        total += stats.mean
        var_sum += stats.variance / stats.n_paths
    return total, math.sqrt(var_sum)


def _check_fail(spec, n_fail):
    if n_fail is not None:
        nf = int(n_fail.item())
        if nf:
            raise NumericalError(f"exact CIR transition failed at level {spec.level}: {nf} transitions "
                                 "exceeded the 1e-8 residual contract")


def merge_triples(parts: np.ndarray) -> np.ndarray:
    """Chan-merge rows of (count, mean, M2) triples, in order."""
    out = np.zeros(3)
    for n_b, m_b, m2_b in parts:
        n_a, m_a, m2_a = out
        if n_b == 0:
            continue
        if n_a == 0:
            out = np.array([n_b, m_b, m2_b])
            continue
        tot = n_a + n_b
        delta = m_b - m_a
        out = np.array([tot, m_a + delta * (n_b / tot), m2_a + m2_b + delta * delta * (n_a * n_b / tot)])
    return out


def _host_if_gloo(t: torch.Tensor, group=None) -> torch.Tensor:
    """gloo reduces host tensors; NCCL keeps them on the device."""
    import torch.distributed as dist

    return t.cpu() if dist.get_backend(group) == "gloo" else t


def allreduce_triples(triples: torch.Tensor, group=None) -> torch.Tensor:
    """Merge per-rank (count, mean, M2) rows across a torch.distributed group.

    Two all-reduces of 2*NSLOT and NSLOT doubles: first (n, n*mean) -> global
    mean mu; then each rank's M2 re-centred on mu (M2_r + n_r (mean_r - mu)^2,
    exact algebra) is summed.  Works for NCCL (CUDA tensors) and gloo (CPU).
    """
    import torch.distributed as dist

    t = _host_if_gloo(triples.to(torch.float64), group)
    n = t[:, 0].clone()
    s1 = torch.stack([n, n * t[:, 1]], dim=1).contiguous()
    dist.all_reduce(s1, group=group)
    n_tot = s1[:, 0]
    mu = torch.where(n_tot > 0, s1[:, 1] / torch.clamp(n_tot, min=1.0), torch.zeros_like(n_tot))
    m2 = (t[:, 2] + n * (t[:, 1] - mu) ** 2).contiguous()
    dist.all_reduce(m2, group=group)
    return torch.stack([n_tot, mu, m2], dim=1)


def _stats_from(level: int, kind: str, triple, seconds: float, draws: float) -> LevelStats:
    n, mean, m2 = (float(x) for x in triple)
    var = m2 / (n - 1.0) if n > 1 else 0.0
    return LevelStats(level=level, kind=kind, mean=mean, variance=var, n_paths=int(n),
                      cost_per_path_seconds=seconds / max(n, 1.0), cost_per_path_draws=float(draws),
                      degenerate=var == 0.0)


def _timed_level(spec, stream, n_pilot, group=None, sides: str = "both"):
    device = dev.require_cuda()
    rank, world = 0, 1
    if group is not None or _dist_ready():
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
    per = n_pilot // world
    extra = n_pilot % world
    lo = rank * per + min(rank, extra)
    cnt = per + (1 if rank < extra else 0)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record()
    stats, _, n_fail = run_level(spec, stream, n_pilot, path_lo=lo, path_count=cnt, device=device, sides=sides)
    stop.record()
    if world > 1:
        import torch.distributed as dist

        stats = allreduce_triples(stats, group)
        if n_fail is not None:  # every rank raises if any rank's transitions failed
            n_fail = _host_if_gloo(n_fail, group)
            dist.all_reduce(n_fail, group=group)
    stop.synchronize()
    _check_fail(spec, n_fail)
    seconds = start.elapsed_time(stop) * 1e-3
    return stats.cpu().numpy(), seconds * world  # device-seconds summed over ranks


def _dist_ready() -> bool:
    try:
        import torch.distributed as dist

        return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
    except Exception:  # pragma: no cover
        return False


def estimate_level(spec: LevelSpec, stream: Pcg32Stream, n_pilot: int, group=None) -> LevelStats:
    """Pilot-run one level: mean/variance plus measured costs (mlmc.py:356-380)."""
    if n_pilot < 100:
        raise ConfigError(f"pilot size must be >= 100, got {n_pilot}")
    stats, seconds = _timed_level(spec, stream, n_pilot, group, sides=_sides_for(spec))
    exact = _is_exact(spec.rv_source)
    if spec.scheme == "cir_exact":
        slot = {"plain": 3 if exact else 4, "two_way": 0 if exact else 1, "four_way": 2}[spec.kind]
    else:
        slot = {"plain": 3 if exact else 4, "two_way": 0 if exact else 1, "four_way": 2}[spec.kind]
    return _stats_from(spec.level, spec.kind, stats[slot], seconds, spec.n_steps_fine)


def estimate_level_suite(spec: LevelSpec, stream: Pcg32Stream, n_pilot: int, group=None) -> dict:
    """Exact two-way, approximate two-way and four-way stats in one pass (mlmc.py:383-411).

    For ``cir_exact`` (where coarse repeats fine) the suite instead holds the
    exact and approximate process statistics and the exact - approximate
    ``correction`` (reproduce.py:293-303).
    """
    if n_pilot < 100:
        raise ConfigError(f"pilot size must be >= 100, got {n_pilot}")
    if _is_exact(spec.rv_source):
        raise ConfigError("suite estimation needs a table source")
    stats, seconds = _timed_level(spec, stream, n_pilot, group)
    return _suite_from(spec, stats, seconds)


def _suite_from(spec: LevelSpec, stats, seconds: float) -> dict:
    draws = spec.n_steps_fine
    if spec.scheme == "cir_exact":
        return {
            "plain_exact": _stats_from(spec.level, "plain", stats[3], seconds, draws),
            "plain_approx": _stats_from(spec.level, "plain", stats[4], seconds, draws),
            "correction": _stats_from(spec.level, "four_way", stats[2], seconds, draws),
        }
    return {
        "two_way_exact": _stats_from(spec.level, "two_way", stats[0], seconds, draws),
        "two_way_approx": _stats_from(spec.level, "two_way", stats[1], seconds, draws),
        "four_way": _stats_from(spec.level, "four_way", stats[2], seconds, draws),
    }


_EVENT_POOL: list = []


def _events(n: int) -> list:
    """n timing events from a pool (creating CUDA events costs host time)."""
    while len(_EVENT_POOL) < n:
        _EVENT_POOL.append(torch.cuda.Event(enable_timing=True))
    return _EVENT_POOL[:n]


def estimate_level_suites(specs: list, streams: list, n_pilot: int, group=None) -> list:
    """``estimate_level_suite`` for every level of a pilot in one pass.

    The levels are launched back to back on the device (no host round trip
    between them), each rank simulating its contiguous share of every
    level's paths; the per-level (count, mean, M2) triples of all levels are
    merged across ranks with ONE pair of all-reduces (NCCL on GPUs) and the
    failure counts with one more, and the host synchronises once.  Results
    equal the per-level calls (same paths, same merge); per-level device
    seconds come from CUDA events between the launches.
    """
    if len(specs) != len(streams):
        raise ConfigError("one stream per level spec")
    if n_pilot < 100:
        raise ConfigError(f"pilot size must be >= 100, got {n_pilot}")
    if any(_is_exact(sp.rv_source) for sp in specs):
        raise ConfigError("suite estimation needs a table source")
    device = dev.require_cuda()
    rank, world = 0, 1
    if group is not None or _dist_ready():
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
    per, extra = divmod(n_pilot, world)
    lo = rank * per + min(rank, extra)
    cnt = per + (1 if rank < extra else 0)
    # one stats block, one workspace and one failure counter for all levels
    # (stream-ordered reuse), timing events from a pool
    allst = torch.empty((len(specs) * NSLOT, 3), dtype=torch.float64, device=device)
    ws = torch.empty(max(_workspace_bytes(sp, cnt, device) for sp in specs), dtype=torch.uint8, device=device)
    has_cir = any(sp.scheme == "cir_exact" for sp in specs)
    n_fail = torch.zeros(1, dtype=torch.int64, device=device) if has_cir else None
    evs = _events(len(specs) + 1)
    evs[0].record()
    for k, (spec, stream) in enumerate(zip(specs, streams)):
        run_level(spec, stream, n_pilot, path_lo=lo, path_count=cnt, device=device,
                  stats_out=allst[k * NSLOT:(k + 1) * NSLOT].view(-1), workspace=ws, n_fail_out=n_fail)
        evs[k + 1].record()
    if world > 1:
        import torch.distributed as dist

        allst = allreduce_triples(allst, group)
        if n_fail is not None:
            n_fail = _host_if_gloo(n_fail, group)
            dist.all_reduce(n_fail, group=group)
    evs[-1].synchronize()
    if n_fail is not None and int(n_fail.item()):
        raise NumericalError(f"exact CIR transition failed: {int(n_fail.item())} transitions exceeded the "
                             "1e-8 residual contract")
    host = allst.cpu().numpy().reshape(len(specs), NSLOT, 3)
    return [_suite_from(spec, host[k], evs[k].elapsed_time(evs[k + 1]) * 1e-3 * world)
            for k, spec in enumerate(specs)]


# ---------------------------------------------------------------------------
# Allocation and speed-up accounting: host arithmetic on per-level scalars,
# restated from mlmc.py:424-550 (out of the hot path; kept for drop-in use).
# ---------------------------------------------------------------------------

@dataclass
class Allocation:
    n_paths: list
    predicted_cost: float
    epsilon: float
    variance_budget_used: float


def _stat_cost(stats: LevelStats, cost_model: str) -> float:
    return stats.cost_per_path_draws if cost_model == "draws" else stats.cost_per_path_seconds


def optimal_allocation(level_stats, epsilon: float, cost_model: str = "draws") -> Allocation:
    """m_l = eps^-1 sqrt(2 T v_l / c_l), T = 2 eps^-2 (sum sqrt(v c))^2 (mlmc.py:436-460)."""
    stats = list(level_stats)
    if not stats:
        raise ConfigError("allocation needs at least one level")
    if epsilon <= 0:
        raise ConfigError("epsilon must be > 0")
    v = np.array([s.variance for s in stats])
    c = np.array([_stat_cost(s, cost_model) for s in stats])
    if np.any(v < 0) or np.any(c <= 0):
        raise ConfigError("variances must be >= 0 and costs > 0")
    total_cost = 2.0 * epsilon**-2 * np.sqrt(v * c).sum() ** 2
    with np.errstate(divide="ignore", invalid="ignore"):
        m_real = epsilon**-1 * np.sqrt(2.0 * total_cost * v / c)
    m = np.maximum(np.ceil(np.nan_to_num(m_real)), 1.0)
    return Allocation([int(x) for x in m], float(total_cost), epsilon, float(np.sum(v / m)))


def optimal_allocation_nested(two_way_stats, four_way_stats, epsilon: float, cost_model: str = "draws"):
    """Cheap and correction allocations of the nested estimator (mlmc.py:463-487)."""
    tw, fw = list(two_way_stats), list(four_way_stats)
    if len(tw) != len(fw) or not tw:
        raise ConfigError("need matching per-level two-way and four-way stats")
    if epsilon <= 0:
        raise ConfigError("epsilon must be > 0")
    v_t = np.array([s.variance for s in tw])
    c_t = np.array([_stat_cost(s, cost_model) for s in tw])
    v_f = np.array([s.variance for s in fw])
    c_f = np.array([_stat_cost(s, cost_model) for s in fw])
    total = 2.0 * epsilon**-2 * (np.sqrt(v_t * c_t) + np.sqrt(v_f * c_f)).sum() ** 2
    with np.errstate(divide="ignore", invalid="ignore"):
        m = np.maximum(np.ceil(epsilon**-1 * np.sqrt(2.0 * total * v_t / c_t)), 1.0)
        mm = np.maximum(np.ceil(np.nan_to_num(epsilon**-1 * np.sqrt(2.0 * total * v_f / c_f))), 1.0)
    cheap = Allocation([int(x) for x in m], float(np.sum(m * c_t)), epsilon, float(np.sum(v_t / m)))
    corr = Allocation([int(x) for x in mm], float(np.sum(mm * c_f)), epsilon, float(np.sum(v_f / mm)))
    return cheap, corr, float(total)


@dataclass
class SpeedupRow:
    name: str
    log2_variance_gap: float
    cost_ratio: float
    speedup: float
    efficiency: float
    paths_ratio_cheap: float
    paths_ratio_correction: float


def speedup_row(name: str, suites: list, cost_ratio: float, level_window=None) -> SpeedupRow:
    """Collapse per-level suites into one savings row (mlmc.py:503-536)."""
    if cost_ratio <= 0:
        raise ConfigError("cost ratio must be > 0")
    gaps = []
    for suite in suites:
        lvl = suite["four_way"].level
        if level_window and not (level_window[0] <= lvl <= level_window[1]):
            continue
        v_hat, v_four = suite["two_way_exact"].variance, suite["four_way"].variance
        if v_hat > 0 and v_four > 0:
            gaps.append(math.log2(v_four / v_hat))
    if not gaps:
        raise ConfigError("no usable levels in window")
    gap = float(np.mean(gaps))
    efficiency = (1.0 + math.sqrt(2.0**gap * (1.0 + cost_ratio))) ** -2
    return SpeedupRow(name, gap, cost_ratio, cost_ratio * efficiency, efficiency,
                      math.sqrt(cost_ratio / (cost_ratio * efficiency)),
                      math.sqrt(2.0**-gap * (1.0 + cost_ratio)))


def speedup_report(pilot_suites: dict, cost_ratios: dict, level_window=None) -> list:
    return [speedup_row(n, s, cost_ratios[n], level_window) for n, s in pilot_suites.items()]

"""Immutable table types (mirroring approxrv/tables.py:27-153) and the shipped tables.

Tables are frozen dataclasses over read-only numpy arrays, exactly as in the
reference, so the device cache in ``_device.table_on_device`` can key on the
buffer.  Reference table objects (``approxrv.tables.*``) are accepted
everywhere by duck typing (``values`` / ``coeffs`` / ``coeffs32`` /
``eval_stacks``).

New here: :class:`SubDyadicTable`, the octave x sub-interval layout of
BASELINE.json config 2 (16 geometrically halving octaves per tail, each split
into 2^sub_bits equal sub-intervals, one degree-m L2 fit per sub-interval).

Shipped tables (``data/tables.npz``) were produced by the reference's own
fitters (``tools/make_tables.py``); fitting is an offline CPU step outside the
hot path.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from functools import cached_property, lru_cache

import numpy as np

from .errors import ConfigError

CONSTRUCTIONS = ("l1", "central", "interior", "rademacher")
_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "tables.npz")


def _frozen_array(a, shape=None, dtype=np.float64) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    if shape is not None and arr.shape != shape:
        raise ConfigError(f"expected array of shape {shape}, got {arr.shape}")
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class ConstantTable:
    """Piecewise-constant quantile approximation on 2^q equal intervals (tables.py:27-48)."""

    q: int
    values: np.ndarray
    construction: str = "l1"

    def __post_init__(self):
        if not 1 <= self.q <= 24:
            raise ConfigError(f"interval exponent q must be in [1, 24], got {self.q}")
        if self.construction not in CONSTRUCTIONS:
            raise ConfigError(f"unknown construction {self.construction!r}")
        object.__setattr__(self, "values", _frozen_array(self.values, (1 << self.q,)))

    @property
    def n_intervals(self) -> int:
        return 1 << self.q

    @cached_property
    def values32(self) -> np.ndarray:
        return _frozen_array(self.values, dtype=np.float32)

    def breakpoints(self) -> np.ndarray:
        return np.linspace(0.0, 1.0, self.n_intervals + 1)


@dataclass(frozen=True)
class DyadicPolyTable:
    """Piecewise polynomial on dyadically decaying intervals (tables.py:51-95).

    ``coeffs`` is coefficient-major (degree+1, K+1); entry 0 is the u = 1/2
    slot, entry k >= 1 covers [2^-(k+1), 2^-k), entry K the singular rest.
    """

    degree: int
    n_intervals: int
    coeffs: np.ndarray
    decay: float = 0.5

    def __post_init__(self):
        if not 1 <= self.degree <= 5:
            raise ConfigError(f"polynomial degree must be in [1, 5], got {self.degree}")
        if not 2 <= self.n_intervals <= 40:
            raise ConfigError(f"interval count must be in [2, 40], got {self.n_intervals}")
        if not 0.0 < self.decay < 1.0:
            raise ConfigError(f"decay rate must be in (0, 1), got {self.decay}")
        object.__setattr__(self, "coeffs", _frozen_array(self.coeffs, (self.degree + 1, self.n_intervals + 1)))

    @cached_property
    def coeffs32(self) -> np.ndarray:
        return _frozen_array(self.coeffs, dtype=np.float32)

    @cached_property
    def natural32(self) -> np.ndarray:
        """(degree+1, K, 1) f32: the same table in the octave x sub-interval
        layout with sub_bits = 0 (used by the fused generator)."""
        return _frozen_array(self.coeffs32[:, 1:, None], dtype=np.float32)

    def interval_bounds(self, k: int) -> tuple[float, float]:
        if k == 0:
            return (0.5, 0.5)
        upper = 0.5 * self.decay ** (k - 1)
        lower = 0.0 if k == self.n_intervals else 0.5 * self.decay**k
        return (lower, upper)


@dataclass(frozen=True)
class SubDyadicTable:
    """Octave x sub-interval table (new layout; BASELINE.json config 2).

    ``coeffs`` (degree+1, K, 2^sub_bits), float64, natural order: octave
    j = 1..K-1 covers [2^-(j+1), 2^-j) split into 2^sub_bits equal
    sub-intervals selected by the top mantissa bits of v = min(u, 1-u);
    octave K is the singular remainder (0, 2^-K), which uses sub-slot 0.
    v = 1/2 evaluates to zero (the reference's u = 1/2 slot).
    """

    degree: int
    n_octaves: int
    sub_bits: int
    coeffs: np.ndarray

    def __post_init__(self):
        if not 1 <= self.degree <= 5:
            raise ConfigError(f"polynomial degree must be in [1, 5], got {self.degree}")
        if not 1 <= self.n_octaves <= 40:
            raise ConfigError(f"octave count must be in [1, 40], got {self.n_octaves}")
        if not 0 <= self.sub_bits <= 5:
            raise ConfigError(f"sub_bits must be in [0, 5], got {self.sub_bits}")
        shape = (self.degree + 1, self.n_octaves, 1 << self.sub_bits)
        object.__setattr__(self, "coeffs", _frozen_array(self.coeffs, shape))

    @property
    def n_sub(self) -> int:
        return 1 << self.sub_bits

    @cached_property
    def coeffs32(self) -> np.ndarray:
        return _frozen_array(self.coeffs, dtype=np.float32)

    @classmethod
    def from_dyadic(cls, table: DyadicPolyTable, sub_bits: int = 0) -> "SubDyadicTable":
        """Replicate a reference dyadic table into the sub-interval layout."""
        nat = np.repeat(np.asarray(table.coeffs)[:, 1:, None], 1 << sub_bits, axis=2)
        return cls(table.degree, table.n_intervals, sub_bits, nat)

    def interval_bounds(self, j: int, s: int) -> tuple[float, float]:
        if j >= self.n_octaves:
            return (0.0, 2.0 ** -self.n_octaves)
        a = 2.0 ** -(j + 1)
        h = a / self.n_sub
        return (a + s * h, a + (s + 1) * h)


@dataclass(frozen=True)
class NcChi2Table:
    """Non-central chi-squared table family (tables.py:98-153), held as its
    evaluation stacks (2, n_knots, degree+1, K+1): upper half at 0, lower at 1."""

    nu: float
    n_knots: int
    degree: int
    n_intervals: int
    eval_stacks: np.ndarray

    def __post_init__(self):
        if not self.nu > 0:
            raise ConfigError(f"nu must be > 0, got {self.nu}")
        if self.n_knots < 2:
            raise ConfigError(f"need at least 2 knots, got {self.n_knots}")
        shape = (2, self.n_knots, self.degree + 1, self.n_intervals + 1)
        object.__setattr__(self, "eval_stacks", _frozen_array(self.eval_stacks, shape))

    @classmethod
    def from_stacks(cls, nu: float, stacks) -> "NcChi2Table":
        s = np.asarray(stacks)
        return cls(float(nu), s.shape[1], s.shape[2] - 1, s.shape[3] - 1, s)

    @classmethod
    def from_reference(cls, table) -> "NcChi2Table":
        return cls.from_stacks(table.nu, table.eval_stacks)

    @property
    def sqrt_y_knots(self) -> np.ndarray:
        return np.linspace(0.0, 1.0, self.n_knots)

    @property
    def lower_stack(self) -> np.ndarray:
        return self.eval_stacks[1]

    @property
    def upper_stack(self) -> np.ndarray:
        return self.eval_stacks[0]


# ---------------------------------------------------------------------------
# Shipped tables
# ---------------------------------------------------------------------------

@lru_cache(maxsize=1)
def _npz() -> dict:
    with np.load(_DATA) as z:
        return {k: z[k] for k in z.files}


def shipped_names() -> list[str]:
    return sorted(k for k in _npz() if not k.endswith("_nu"))


@lru_cache(maxsize=None)
def load_table(name: str):
    """A shipped table by name (see tools/make_tables.py for provenance)."""
    z = _npz()
    if name not in z:
        raise ConfigError(f"unknown shipped table {name!r}; have {shipped_names()}")
    a = z[name]
    if name.startswith("constant_q"):
        q = int(np.log2(a.size))
        return ConstantTable(q, a, "l1")
    if name.startswith("dyadic_"):
        return DyadicPolyTable(a.shape[0] - 1, a.shape[1] - 1, a)
    if name.startswith("subdyadic_"):
        return SubDyadicTable(a.shape[0] - 1, a.shape[1], int(np.log2(a.shape[2])), a)
    if name.startswith("ncchi2_"):
        nu = float(z[name.replace("_stacks", "_nu")])
        return NcChi2Table.from_stacks(nu, a)
    raise ConfigError(f"cannot interpret shipped table {name!r}")

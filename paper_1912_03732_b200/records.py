"""Value types and exceptions of the public API.

Field names, shapes and dtypes are those of the reference package so a
caller of `sboxeval` can switch imports:
  SBox                 pkg/src/sboxeval/sbox.py:51-91
  PolarityTruthTable   pkg/src/sboxeval/sbox.py:128-142
  WalshSpectrum        pkg/src/sboxeval/walsh.py:32-44
  ColumnMaxima         pkg/src/sboxeval/walsh.py:47-53
  NonlinearityResult   pkg/src/sboxeval/nonlinearity.py:29-33
  ColumnPartition      pkg/src/sboxeval/parallel.py:30-35
  MemoryBudgetError    pkg/src/sboxeval/memory.py:16-25
  SizeCapError         pkg/src/sboxeval/nonlinearity.py:25-26
  SBoxFormatError      pkg/src/sboxeval/sbox.py:41-48
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MAX_BITS = 24  # n, m range of the reference (sbox.py:18)


class MemoryBudgetError(RuntimeError):
    """A materialised spectrum would exceed the caller's byte budget."""

    def __init__(self, required: int, budget: int):
        self.required = required
        self.budget = budget
        super().__init__(
            f"spectrum storage needs {required:,} bytes but the budget is {budget:,} bytes"
        )


class SizeCapError(ValueError):
    """The exhaustive affine-distance search only runs on small boxes."""


class SBoxFormatError(ValueError):
    """Malformed .sbox text; `line` is the 1-based offending line (or None)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


@dataclass(frozen=True, eq=False)
class SBox:
    """n-bit -> m-bit lookup table; `table` is a read-only uint32 array of 2^n words."""

    n: int
    m: int
    table: np.ndarray = field(repr=False)

    def __post_init__(self):
        for name, bits in (("n", self.n), ("m", self.m)):
            if not 1 <= bits <= MAX_BITS:
                raise ValueError(f"{name} must be in 1..{MAX_BITS}, got {bits}")
        tab = np.ascontiguousarray(self.table, dtype=np.uint32)
        size = 1 << self.n
        if tab.shape != (size,):
            raise ValueError(f"table must have {size} entries, got {tab.size}")
        limit = 1 << self.m
        if tab.size and int(tab.max()) >= limit:
            pos = int(np.flatnonzero(tab >= limit)[0])
            raise ValueError(
                f"entry {int(tab[pos])} at index {pos} does not fit in {self.m} bits"
            )
        tab.setflags(write=False)
        object.__setattr__(self, "table", tab)

    def __eq__(self, other) -> bool:
        if not isinstance(other, SBox):
            return NotImplemented
        return (self.n, self.m) == (other.n, other.m) and np.array_equal(self.table, other.table)

    __hash__ = object.__hash__

    def __len__(self) -> int:
        return 1 << self.n

    def is_bijective(self) -> bool:
        return self.n == self.m and np.unique(self.table).size == (1 << self.n)


@dataclass(frozen=True)
class PolarityTruthTable:
    """Mask-major (2^m - 1) x 2^n int32 matrix: rows[v-1][x] = (-1)^{g_v(x)}."""

    n: int
    m: int
    rows: np.ndarray = field(repr=False)

    def row_count(self) -> int:
        return (1 << self.m) - 1


@dataclass(frozen=True)
class WalshSpectrum:
    """Mask-major spectrum: rows[v-1][u] = W(u, v), v = 1 .. 2^m - 1 (int32)."""

    n: int
    m: int
    rows: np.ndarray = field(repr=False)

    def value(self, u: int, v: int) -> int:
        if v == 0:
            # the all-zero mask is analytic: W(u, 0) = 2^n at u = 0, else 0
            return (1 << self.n) if u == 0 else 0
        return int(self.rows[v - 1, u])


@dataclass(frozen=True)
class ColumnMaxima:
    """Per-component nonlinearities: values[v-1] = (2^n - max_u |W(u,v)|) / 2 (int64)."""

    n: int
    m: int
    values: np.ndarray = field(repr=False)


@dataclass(frozen=True)
class NonlinearityResult:
    value: int
    argmin_v: int  # smallest output mask achieving the minimum
    method: str


@dataclass(frozen=True)
class ColumnPartition:
    """Disjoint ordered half-open mask ranges covering {1, ..., total}."""

    ranges: tuple[tuple[int, int], ...]
    worker_count: int

"""Byte budgets and live-allocation accounting for spectrum storage.

Contract of the reference's memory module (pkg/src/sboxeval/memory.py:16-84)
and memory_estimate (pkg/src/sboxeval/sbox.py:165-183): every call that would
materialise a spectrum checks the caller's `max_bytes` first and raises
MemoryBudgetError; the process-wide `spectrum_allocations` tracker records
what is live while a transform runs (tests read its peak).

On the GPU the stream (fused) path keeps no spectrum at all for n <= 16 --
the component lives in one SM's shared memory -- so it charges nothing; for
n >= 17 it charges the L2-sized device scratch of the multi-pass transform.
Retain mode charges the materialised matrix, as in the reference.
"""
from __future__ import annotations

import os
import threading
from contextlib import contextmanager

from .records import MemoryBudgetError


class AllocationTracker:
    """Thread-safe counter of live spectrum bytes and their high-water mark."""

    def __init__(self) -> None:
        self._mu = threading.Lock()
        self._live = 0
        self._high = 0

    def charge(self, nbytes: int) -> None:
        with self._mu:
            self._live += nbytes
            self._high = max(self._high, self._live)

    def release(self, nbytes: int) -> None:
        with self._mu:
            self._live -= nbytes

    def reset_peak(self) -> None:
        with self._mu:
            self._high = self._live

    @property
    def current_bytes(self) -> int:
        return self._live

    @property
    def peak_bytes(self) -> int:
        return self._high


spectrum_allocations = AllocationTracker()


@contextmanager
def charged(nbytes: int):
    """Charge `nbytes` to the tracker for the duration of a block."""
    spectrum_allocations.charge(nbytes)
    try:
        yield
    finally:
        spectrum_allocations.release(nbytes)


def check_budget(required: int, max_bytes: int | None) -> None:
    if max_bytes is not None and required > max_bytes:
        raise MemoryBudgetError(required, max_bytes)


def physical_memory_bytes() -> int | None:
    try:
        return os.sysconf("SC_PHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError, AttributeError):
        return None


def default_budget() -> int | None:
    """75% of physical RAM, the reference's default (memory.py:79-84)."""
    total = physical_memory_bytes()
    return None if total is None else (total * 3) // 4


def memory_estimate(n: int, m: int, element_width: int = 4, mode: str = "retain",
                    workers: int = 1) -> int:
    """Spectrum + maxima bytes an evaluation needs (sbox.py:165-183 formula).

    retain: the full (2^m - 1) x 2^n matrix; stream: one column per worker
    plus a spare; both plus a 2^m-entry maxima array.
    """
    maxima = (1 << m) * element_width
    if mode == "retain":
        return ((1 << m) - 1) * (1 << n) * element_width + maxima
    if mode == "stream":
        return (workers + 1) * (1 << n) * element_width + maxima
    raise ValueError(f"mode must be 'retain' or 'stream', got {mode!r}")

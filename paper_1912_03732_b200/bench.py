"""Benchmark harness over the GPU pipelines.

Same contract as the reference's harness (pkg/src/sboxeval/bench.py:32-239):
  * one BenchRecord per (method, workers), holding every repetition's
    end-to-end wall time and its transform-only time (the pipeline's
    `timings["transform_s"]`, which here brackets the kernels with a device
    synchronisation);
  * verify-before-time: a warm-up run and every timed run must reproduce the
    single-worker fused reference (value, and the spectrum when retained),
    otherwise BenchVerificationError -- a wrong answer is never a data point;
  * `speedup_report` within each (n, m) group, and a CSV round trip with the
    reference's header.
"""
from __future__ import annotations

import csv
import io
import statistics
import time
from dataclasses import dataclass, field
from typing import IO, Iterable, Sequence

import numpy as np

from .records import NonlinearityResult, SBox, WalshSpectrum
from .nonlinearity import nonlinearity_bruteforce, nonlinearity_from_maxima, nonlinearity_from_spectrum
from .parallel import fwht_parallel
from .walsh import fwht_fused, fwht_rowmajor, fwht_transposed

CSV_HEADER = ("method", "n", "m", "workers", "repetitions", "mean_ms", "stddev_ms",
              "transform_only_mean_ms")


class BenchVerificationError(RuntimeError):
    """A timed run disagreed with the reference result."""


@dataclass
class BenchRecord:
    method: str
    n: int
    m: int
    workers: int
    repetitions: int
    wall_times: list = field(default_factory=list)       # ms, end to end
    transform_times: list = field(default_factory=list)  # ms

    @property
    def mean_ms(self) -> float:
        return statistics.fmean(self.wall_times)

    @property
    def stddev_ms(self) -> float:
        return statistics.pstdev(self.wall_times)

    @property
    def transform_only_mean_ms(self) -> float:
        return statistics.fmean(self.transform_times)

    def sort_key(self) -> tuple:
        return (self.n, self.m, self.method, self.workers)


@dataclass(frozen=True)
class SpeedupRow:
    n: int
    m: int
    method: str
    workers: int
    ratio: float


def _spectral(method, reduce_fn):
    def run(s, workers, mode, budget, timings):
        spec = method(s, budget, timings)
        return reduce_fn(spec, method.__name__.replace("fwht_", "")), spec
    return run


def _run_fused(s, workers, mode, budget, timings):
    spec, cm = fwht_fused(s, mode=mode, max_bytes=budget, timings=timings)
    return nonlinearity_from_maxima(cm, "fused"), spec


def _run_parallel(s, workers, mode, budget, timings):
    spec, cm = fwht_parallel(s, workers=workers, mode=mode, max_bytes=budget, timings=timings)
    return nonlinearity_from_maxima(cm, "parallel"), spec


def _run_brute(s, workers, mode, budget, timings):
    return nonlinearity_bruteforce(s), None


_PIPELINES = {
    "rowmajor": _spectral(fwht_rowmajor, nonlinearity_from_spectrum),
    "transposed": _spectral(fwht_transposed, nonlinearity_from_spectrum),
    "fused": _run_fused,
    "parallel": _run_parallel,
    "bruteforce": _run_brute,
}


def _timed(s: SBox, method: str, workers: int, mode: str, budget: int | None
           ) -> tuple[NonlinearityResult, WalshSpectrum | None, float, float]:
    if method not in _PIPELINES:
        raise ValueError(f"unknown method {method!r}")
    timings: dict = {}
    t0 = time.perf_counter()
    result, spec = _PIPELINES[method](s, workers, mode, budget, timings)
    wall_ms = (time.perf_counter() - t0) * 1e3
    return result, spec, wall_ms, timings.get("transform_s", wall_ms / 1e3) * 1e3


def _check(result: NonlinearityResult, spec: WalshSpectrum | None, want_value: int,
           want_rows: np.ndarray | None, method: str, workers: int) -> None:
    if result.value != want_value:
        raise BenchVerificationError(
            f"{method} (workers={workers}) returned {result.value}, reference says {want_value}")
    if spec is not None and want_rows is not None and not np.array_equal(spec.rows, want_rows):
        raise BenchVerificationError(f"{method} (workers={workers}) spectrum differs from reference")


def run_benchmark(s: SBox, methods: Iterable[str], worker_counts: Sequence[int] = (1,),
                  repetitions: int = 5, mode: str = "retain",
                  max_bytes: int | None = None) -> list[BenchRecord]:
    """Time each method (parallel once per worker count) after a verified warm-up."""
    if repetitions < 1:
        raise ValueError(f"repetitions must be >= 1, got {repetitions}")
    ref_spec, ref_cm = fwht_fused(s, mode=mode, max_bytes=max_bytes)
    want_value = nonlinearity_from_maxima(ref_cm).value
    want_rows = None if ref_spec is None else ref_spec.rows
    records = []
    for method in sorted(set(methods)):
        for workers in (list(worker_counts) if method == "parallel" else [1]):
            rec = BenchRecord(method, s.n, s.m, workers, repetitions)
            for rep in range(repetitions + 1):  # rep 0 = warm-up, verified but not recorded
                result, spec, wall_ms, tr_ms = _timed(s, method, workers, mode, max_bytes)
                _check(result, spec, want_value, want_rows, method, workers)
                if rep:
                    rec.wall_times.append(wall_ms)
                    rec.transform_times.append(tr_ms)
            records.append(rec)
    return sorted(records, key=BenchRecord.sort_key)


def speedup_report(records: Sequence[BenchRecord], baseline_method: str) -> list[SpeedupRow]:
    """baseline mean / record mean within each (n, m) group (higher = faster)."""
    ordered = sorted(records, key=BenchRecord.sort_key)
    base: dict = {}
    for r in ordered:
        if r.method == baseline_method:
            base.setdefault((r.n, r.m), r)
    missing = sorted({(r.n, r.m) for r in ordered} - set(base))
    if missing:
        raise ValueError(f"baseline method {baseline_method!r} not in records for size(s) {missing}")
    return [SpeedupRow(r.n, r.m, r.method, r.workers, base[(r.n, r.m)].mean_ms / r.mean_ms)
            for r in ordered]


def write_csv(records: Sequence[BenchRecord], stream: IO[str]) -> None:
    out = csv.writer(stream, lineterminator="\n")
    out.writerow(CSV_HEADER)
    for r in sorted(records, key=BenchRecord.sort_key):
        out.writerow([r.method, r.n, r.m, r.workers, r.repetitions, repr(r.mean_ms),
                      repr(r.stddev_ms), repr(r.transform_only_mean_ms)])


_CSV_TYPES = {"method": str, "n": int, "m": int, "workers": int, "repetitions": int,
              "mean_ms": float, "stddev_ms": float, "transform_only_mean_ms": float}


def read_csv(stream: IO[str] | str) -> list[dict]:
    """Inverse of write_csv: typed row dicts."""
    src = io.StringIO(stream) if isinstance(stream, str) else stream
    return [{k: _CSV_TYPES[k](row[k]) for k in CSV_HEADER} for row in csv.DictReader(src)]

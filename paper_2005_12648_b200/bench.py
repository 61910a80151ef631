"""Benchmark harness on the device (mirror of ``parmerge.bench``, bench.py:1-345).

Same grid, records, derived tables and CSV schema as the reference harness --
``method,threads,elem_bytes,size,split,mean_ns,min_ns,max_ns`` and the
median-quality study's ``t,size,rel_diff_findmedian`` -- so result files of
both sides load into the same tools (``plots/``).  The differences are where
the work runs:

* every method name maps to this package's entry point of the same name
  (``seq-rotation`` -> ``seq_merge_rotation``, ``srecpar-cs`` ->
  ``merge_srecpar(shift_kind="circular")`` ...), all of which merge on the GPU;
* inputs are generated on the host with the reference's generator
  (``generate_input``, bench.py:110-146), uploaded once per cell and restored
  on the device before every repetition (outside the timed region);
* a repetition is timed with ``time.perf_counter_ns`` around the call plus a
  device synchronisation, i.e. what a caller waits for (bench.py:196-207
  times the call the same way on the CPU);
* validation compares the merged keys with a device sort of the input.
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass, replace

import numpy as np

from .median import find_median, find_median_optimal
from .records import KeyedArray, MergeJob
from .seqmerge import seq_merge_buffered, seq_merge_rotation
from .shift import CIRCULAR, LINEAR
from .soptmov import merge_soptmov
from .srecpar import merge_srecpar
from .workloads import generate_input as _generate_host

METHODS = ("seq-rotation", "seq-buffered", "soptmov", "srecpar-ls", "srecpar-cs")
SEQ_METHODS = ("seq-rotation", "seq-buffered")
DEFAULT_SIZES = tuple(2**k for k in range(2, 15))
DEFAULT_ELEM_BYTES = (4, 64, 512, 1024, 16384, 65540)
DEFAULT_SPLITS = (0.25, 0.5, 0.75)
DEFAULT_THREADS = (8, 16)
QUALITY_THREADS = (2, 4, 8, 16)

RECORD_HEADER = "method,threads,elem_bytes,size,split,mean_ns,min_ns,max_ns"
QUALITY_HEADER = "t,size,rel_diff_findmedian"


class ValidationFailure(Exception):
    """A merge under measurement produced an unsorted or altered key multiset."""


class ConfigError(Exception):
    """The benchmark configuration is inconsistent."""


@dataclass(frozen=True)
class BenchConfig:
    """One measurement campaign (bench.py:41-80): the grid plus run controls."""

    sizes: tuple[int, ...] = DEFAULT_SIZES
    elem_bytes: tuple[int, ...] = DEFAULT_ELEM_BYTES
    splits: tuple[float, ...] = DEFAULT_SPLITS
    methods: tuple[str, ...] = METHODS
    threads: tuple[int, ...] = DEFAULT_THREADS
    reps: int = 50
    seed: int = 1
    out: str | None = None
    max_bytes: int | None = 2**31
    device: str = "cuda"

    def validate(self) -> "BenchConfig":
        """Reject inconsistent grids with ConfigError; splits are quantised to 2 decimals."""
        problems = []
        if any(s < 0 for s in self.sizes):
            problems.append("sizes must be >= 0")
        if any(eb < 4 for eb in self.elem_bytes):
            problems.append("elem_bytes must be >= 4")
        if any(not 0.0 < sp < 1.0 for sp in self.splits):
            problems.append("splits must lie in the open interval (0, 1)")
        if self.reps < 1:
            problems.append("reps must be >= 1")
        bad = [m for m in self.methods if m not in METHODS]
        if bad:
            problems.append(f"unknown methods {bad}; choose from {METHODS}")
        if any(t < 1 or (t & (t - 1)) for t in self.threads):
            problems.append("thread counts must be powers of two >= 1")
        if self.device != "cuda":
            problems.append(f"device must be 'cuda' (this build has no CPU path), got {self.device!r}")
        if problems:
            raise ConfigError(problems[0])
        # the CSV keeps two decimals: round now so written records read back equal
        q = tuple(round(sp, 2) for sp in self.splits)
        if any(not 0.0 < sp < 1.0 for sp in q):
            raise ConfigError("splits must stay inside (0, 1) at 2-decimal precision")
        if len(set(q)) != len(q):
            raise ConfigError("splits collide after 2-decimal rounding")
        return replace(self, splits=q)


@dataclass(frozen=True)
class BenchRecord:
    """One measured grid cell, nanoseconds aggregated over the repetitions."""

    method: str
    threads: int
    elem_bytes: int
    size: int
    split: float
    mean_ns: float
    min_ns: float
    max_ns: float

    def __post_init__(self):
        if not (self.min_ns <= self.mean_ns <= self.max_ns):
            raise ValueError("need min_ns <= mean_ns <= max_ns")


@dataclass(frozen=True)
class SpeedupRow:
    method: str
    threads: int
    elem_bytes: int
    size: int
    speedup: float


@dataclass(frozen=True)
class QualityRow:
    t: int
    size: int
    rel_diff: float


def generate_input(size: int, split: float, seed: int, elem_bytes: int = 4) -> tuple[KeyedArray, int]:
    """The reference's random-walk runs (bench.py:110-146) as a device KeyedArray + middle."""
    keys, payload, middle = _generate_host(size, split, seed, elem_bytes)
    return KeyedArray(keys, payload if payload.shape[1] else None), middle


def _method_call(name: str):
    calls = {
        "seq-rotation": lambda arr, job, t: seq_merge_rotation(arr, job),
        "seq-buffered": lambda arr, job, t: seq_merge_buffered(arr, job),
        "soptmov": lambda arr, job, t: merge_soptmov(arr, job, t),
        "srecpar-ls": lambda arr, job, t: merge_srecpar(arr, job, t, shift_kind=LINEAR),
        "srecpar-cs": lambda arr, job, t: merge_srecpar(arr, job, t, shift_kind=CIRCULAR),
    }
    if name not in calls:
        raise ConfigError(f"unknown method {name!r}")
    return calls[name]


def threads_for(method: str, config: BenchConfig) -> tuple[int, ...]:
    """Sequential methods run once with t = 1; the parallel ones once per worker count."""
    return (1,) if method in SEQ_METHODS else tuple(config.threads)


def iter_cells(config: BenchConfig):
    """(method, threads, elem_bytes, size, split) in emission order, skipping cells over max_bytes."""
    for method in config.methods:
        for t in threads_for(method, config):
            for eb in config.elem_bytes:
                for size in config.sizes:
                    if config.max_bytes is not None and size * eb > config.max_bytes:
                        continue
                    for split in config.splits:
                        yield method, t, eb, size, split


def run_grid(config: BenchConfig, *, validate_only: bool = False, progress=None) -> list[BenchRecord]:
    """Measure every cell: restore the input, merge on the device, verify, aggregate.

    One warm-up repetition per cell is discarded; an unsorted result or a
    changed key multiset raises ValidationFailure naming the cell.
    """
    import torch

    config = config.validate()
    out = []
    for method, t, eb, size, split in iter_cells(config):
        label = f"{method} t={t} elem_bytes={eb} size={size} split={split:.2f}"
        arr, middle = generate_input(size, split, config.seed, eb)
        pristine_k = arr.keys.clone()
        pristine_p = arr.payload.clone()
        want = torch.sort(pristine_k).values
        job = MergeJob(0, middle, size)
        call = _method_call(method)
        reps = 1 if validate_only else config.reps
        samples = []
        for rep in range(reps + 1):
            arr.keys.copy_(pristine_k)
            if pristine_p.shape[1]:
                arr.payload.copy_(pristine_p)
            torch.cuda.synchronize()
            t0 = time.perf_counter_ns()
            call(arr, job, t)
            torch.cuda.synchronize()
            dt = time.perf_counter_ns() - t0
            if not torch.equal(arr.keys, want):
                raise ValidationFailure(f"unsorted or corrupted output in cell [{label}]")
            if rep:
                samples.append(dt)
            if validate_only:
                break
        if progress is not None:
            progress(label)
        if not validate_only:
            out.append(BenchRecord(method, t, eb, size, split, mean_ns=float(np.mean(samples)),
                                   min_ns=float(min(samples)), max_ns=float(max(samples))))
    return out


def speedup_table(records: list[BenchRecord], baseline_method: str) -> list[SpeedupRow]:
    """baseline mean / method mean per (elem_bytes, size, split), averaged over splits.

    Every cell present must have a baseline record (ConfigError otherwise).
    """
    base = {(r.elem_bytes, r.size, r.split): r.mean_ns for r in records if r.method == baseline_method}
    if not base:
        raise ConfigError(f"baseline method {baseline_method!r} has no records")
    ratios: dict[tuple, list[float]] = {}
    for r in records:
        cell = (r.elem_bytes, r.size, r.split)
        if cell not in base:
            raise ConfigError(f"baseline {baseline_method!r} missing cell elem_bytes={r.elem_bytes} "
                              f"size={r.size} split={r.split:.2f}")
        ratios.setdefault((r.method, r.threads, r.elem_bytes, r.size), []).append(base[cell] / r.mean_ns)
    return [SpeedupRow(m, t, eb, size, float(np.mean(v))) for (m, t, eb, size), v in ratios.items()]


def largest_leaf_pair(keys, middle: int, t: int, median_fn) -> int:
    """Largest of the t leaf pairs left by log2(t) levels of recursive division with median_fn."""
    if t < 1 or (t & (t - 1)):
        raise ConfigError("t must be a power of two >= 1")
    level = [(keys[:middle], keys[middle:])]
    while len(level) < t:
        split_level = []
        for a, b in level:
            p_a, p_b = median_fn(a, b)
            split_level += [(a[:p_a], b[:p_b]), (a[p_a:], b[p_b:])]
        level = split_level
    return max(len(a) + len(b) for a, b in level)


def median_quality_study(config: BenchConfig) -> list[QualityRow]:
    """Worst leaf of find_median vs find_median_optimal, relative, averaged over splits.

    Both searches run on the device over the same generated runs (bench.py's
    study, Fig. 5 of the paper): (max_heuristic - max_optimal) / max_optimal.
    """
    config = config.validate()
    rows = []
    for t in QUALITY_THREADS:
        for size in config.sizes:
            diffs = []
            for split in config.splits:
                arr, middle = generate_input(size, split, config.seed)
                heur = largest_leaf_pair(arr.keys, middle, t, find_median)
                best = largest_leaf_pair(arr.keys, middle, t, find_median_optimal)
                diffs.append(0.0 if best == 0 else (heur - best) / best)
            rows.append(QualityRow(t, size, float(np.mean(diffs))))
    return rows


def write_records_csv(path, records: list[BenchRecord]) -> None:
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(RECORD_HEADER.split(","))
        w.writerows([r.method, r.threads, r.elem_bytes, r.size, f"{r.split:.2f}", repr(r.mean_ns), repr(r.min_ns),
                     repr(r.max_ns)] for r in records)


def read_records_csv(path) -> list[BenchRecord]:
    with open(path, encoding="utf-8", newline="") as fh:
        rows = list(csv.reader(fh))
    if not rows or rows[0] != RECORD_HEADER.split(","):
        raise ConfigError(f"unexpected CSV header {rows[0] if rows else None}")
    return [BenchRecord(m, int(t), int(eb), int(sz), float(sp), float(a), float(lo), float(hi))
            for m, t, eb, sz, sp, a, lo, hi in rows[1:]]


def write_quality_csv(path, rows: list[QualityRow]) -> None:
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(QUALITY_HEADER.split(","))
        w.writerows([r.t, r.size, repr(r.rel_diff)] for r in rows)

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

import collections
import csv
import itertools
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
    """A measured merge left unsorted keys or changed the key multiset."""


class ConfigError(Exception):
    """An inconsistent measurement grid."""


def _is_pow2(t: int) -> bool:
    return t >= 1 and t & (t - 1) == 0


@dataclass(frozen=True)
class BenchConfig:
    """A measurement campaign: the grid (sizes x widths x splits x methods x threads) plus controls."""

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
        """ConfigError on the first inconsistency; returns a copy with splits quantised to 2 decimals."""
        unknown = [m for m in self.methods if m not in METHODS]
        checks = (
            (all(x >= 0 for x in self.sizes), "sizes must be >= 0"),
            (all(x >= 4 for x in self.elem_bytes), "elem_bytes must be >= 4"),
            (all(0.0 < x < 1.0 for x in self.splits), "splits must lie in the open interval (0, 1)"),
            (self.reps >= 1, "reps must be >= 1"),
            (not unknown, f"unknown methods {unknown}; choose from {METHODS}"),
            (all(map(_is_pow2, self.threads)), "thread counts must be powers of two >= 1"),
            (self.device == "cuda", f"device must be 'cuda' (this build has no CPU path), got {self.device!r}"),
        )
        for ok, why in checks:
            if not ok:
                raise ConfigError(why)
        # the CSV keeps two decimals: quantise now so written records read back equal
        q = tuple(round(x, 2) for x in self.splits)
        if not all(0.0 < x < 1.0 for x in q):
            raise ConfigError("splits must stay inside (0, 1) at 2-decimal precision")
        if len(set(q)) < len(q):
            raise ConfigError("splits collide after 2-decimal rounding")
        return replace(self, splits=q)


@dataclass(frozen=True)
class BenchRecord:
    """One grid cell's timing (nanoseconds over the repetitions)."""

    method: str
    threads: int
    elem_bytes: int
    size: int
    split: float
    mean_ns: float
    min_ns: float
    max_ns: float

    def __post_init__(self):
        if self.min_ns > self.mean_ns or self.mean_ns > self.max_ns:
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
    """The reference harness's random-walk runs (bench.py:110-146), as a device KeyedArray, and the middle."""
    keys, payload, middle = _generate_host(size, split, seed, elem_bytes)
    return KeyedArray(keys, payload if payload.shape[1] else None), middle


# method name -> device call (arr, job, t); the sequential ones ignore t
_CALLS = {
    "seq-rotation": lambda arr, job, t: seq_merge_rotation(arr, job),
    "seq-buffered": lambda arr, job, t: seq_merge_buffered(arr, job),
    "soptmov": lambda arr, job, t: merge_soptmov(arr, job, t),
    "srecpar-ls": lambda arr, job, t: merge_srecpar(arr, job, t, shift_kind=LINEAR),
    "srecpar-cs": lambda arr, job, t: merge_srecpar(arr, job, t, shift_kind=CIRCULAR),
}


def threads_for(method: str, config: BenchConfig) -> tuple[int, ...]:
    """t = 1 for the sequential methods, every configured worker count for the parallel ones."""
    return (1,) if method in SEQ_METHODS else tuple(config.threads)


def iter_cells(config: BenchConfig):
    """Grid cells (method, threads, elem_bytes, size, split) in emission order, within max_bytes."""
    cap = config.max_bytes
    for method in config.methods:
        for t, eb, size, split in itertools.product(threads_for(method, config), config.elem_bytes, config.sizes,
                                                     config.splits):
            if cap is None or size * eb <= cap:
                yield method, t, eb, size, split


def _time_cell(call, arr, job, t, pristine, want, reps: int, label: str) -> list[int]:
    import torch

    pk, pp = pristine
    samples = []
    for rep in range(reps + 1):  # repetition 0 warms up
        arr.keys.copy_(pk)
        if pp.shape[1]:
            arr.payload.copy_(pp)
        torch.cuda.synchronize()
        t0 = time.perf_counter_ns()
        call(arr, job, t)
        torch.cuda.synchronize()
        dt = time.perf_counter_ns() - t0
        if not torch.equal(arr.keys, want):
            raise ValidationFailure(f"unsorted or corrupted output in cell [{label}]")
        samples.append(dt)
    return samples[1:]


def run_grid(config: BenchConfig, *, validate_only: bool = False, progress=None) -> list[BenchRecord]:
    """Measure every cell on the device: restore the input, merge, check against a device sort.

    validate_only runs each cell once and returns no records.
    """
    import torch

    config = config.validate()
    records = []
    for method, t, eb, size, split in iter_cells(config):
        label = f"{method} t={t} elem_bytes={eb} size={size} split={split:.2f}"
        arr, middle = generate_input(size, split, config.seed, eb)
        pristine = (arr.keys.clone(), arr.payload.clone())
        want = torch.sort(pristine[0]).values
        samples = _time_cell(_CALLS[method], arr, MergeJob(0, middle, size), t, pristine, want,
                             0 if validate_only else config.reps, label)
        if progress is not None:
            progress(label)
        if samples:
            records.append(BenchRecord(method, t, eb, size, split, mean_ns=float(np.mean(samples)),
                                       min_ns=float(min(samples)), max_ns=float(max(samples))))
    return records


def speedup_table(records: list[BenchRecord], baseline_method: str) -> list[SpeedupRow]:
    """Per (method, threads, elem_bytes, size): mean over splits of baseline_ns / method_ns.

    Every cell needs a baseline record with the same (elem_bytes, size, split).
    """
    base = {(r.elem_bytes, r.size, r.split): r.mean_ns for r in records if r.method == baseline_method}
    if not base:
        raise ConfigError(f"baseline method {baseline_method!r} has no records")
    groups: dict[tuple, list[float]] = collections.defaultdict(list)
    for r in records:
        ref = base.get((r.elem_bytes, r.size, r.split))
        if ref is None:
            raise ConfigError(f"baseline {baseline_method!r} missing cell elem_bytes={r.elem_bytes} "
                              f"size={r.size} split={r.split:.2f}")
        groups[(r.method, r.threads, r.elem_bytes, r.size)].append(ref / r.mean_ns)
    return [SpeedupRow(*key, speedup=float(np.mean(v))) for key, v in groups.items()]


def largest_leaf_pair(keys, middle: int, t: int, median_fn) -> int:
    """Size of the largest of the t leaf pairs that log2(t) levels of division by median_fn leave."""
    if not _is_pow2(t):
        raise ConfigError("t must be a power of two >= 1")
    pairs = [(keys[:middle], keys[middle:])]
    for _ in range(t.bit_length() - 1):
        pairs = [half for a, b in pairs for half in _halves(a, b, median_fn)]
    return max(len(a) + len(b) for a, b in pairs)


def _halves(a, b, median_fn):
    p_a, p_b = median_fn(a, b)
    return (a[:p_a], b[:p_b]), (a[p_a:], b[p_b:])


def median_quality_study(config: BenchConfig) -> list[QualityRow]:
    """Fig. 5 study on the device: (worst leaf of find_median - worst of find_median_optimal) / the
    latter, averaged over the splits, for t in QUALITY_THREADS and every size."""
    config = config.validate()

    def rel(size, split, t):
        arr, middle = generate_input(size, split, config.seed)
        best = largest_leaf_pair(arr.keys, middle, t, find_median_optimal)
        return 0.0 if best == 0 else (largest_leaf_pair(arr.keys, middle, t, find_median) - best) / best

    return [QualityRow(t, size, float(np.mean([rel(size, sp, t) for sp in config.splits])))
            for t in QUALITY_THREADS for size in config.sizes]


_RECORD_FIELDS = RECORD_HEADER.split(",")


def write_records_csv(path, records: list[BenchRecord]) -> None:
    with open(path, "w", encoding="utf-8", newline="") as fh:
        out = csv.DictWriter(fh, _RECORD_FIELDS, lineterminator="\n")
        out.writeheader()
        for r in records:
            row = {f: getattr(r, f) for f in _RECORD_FIELDS}
            row.update(split=f"{r.split:.2f}", mean_ns=repr(r.mean_ns), min_ns=repr(r.min_ns), max_ns=repr(r.max_ns))
            out.writerow(row)


def read_records_csv(path) -> list[BenchRecord]:
    with open(path, encoding="utf-8", newline="") as fh:
        rd = csv.reader(fh)
        header = next(rd, None)
        if header != _RECORD_FIELDS:
            raise ConfigError(f"unexpected CSV header {header}")
        casts = (str, int, int, int, float, float, float, float)
        return [BenchRecord(*(c(v) for c, v in zip(casts, row))) for row in rd]


def write_quality_csv(path, rows: list[QualityRow]) -> None:
    with open(path, "w", encoding="utf-8", newline="") as fh:
        fh.write(QUALITY_HEADER + "\n")
        fh.writelines(f"{r.t},{r.size},{r.rel_diff!r}\n" for r in rows)

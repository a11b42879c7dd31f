"""Benchmark protocol for kernel variants, borrowed from the reference's
autoselect (autoselect.py:75-115): every
candidate runs 2m+1 times, candidates interleaved round-robin so clock drift
spreads over all of them, and each reports the mean of its own LAST m runs
(the first m+1 absorb warm-up).  There is no runtime dispatch: this measures
plan / build variants of the one fused kernel family, it does not pick
engines (the north star excludes multi-backend dispatch).

Timing is on the device: a CUDA event pair around each execution on the
current stream (`cuda_timer`), or any injected clock (tests use a scripted
one, like the reference's tests/test_autoselect.py:9-27).
"""

from __future__ import annotations

import os
import statistics
from contextlib import contextmanager
from dataclasses import dataclass, field

DEFAULT_M = 5  # autoselect.py:27


@dataclass
class BenchEntry:
    name: str
    mean_seconds: float
    runs: list = field(default_factory=list)


@dataclass
class BenchReport:
    entries: list = field(default_factory=list)

    @property
    def best(self) -> BenchEntry:
        return min(self.entries, key=lambda e: e.mean_seconds)

    def to_text(self) -> str:
        lines = [f"candidate={e.name} mean_seconds={e.mean_seconds:.9e} runs={len(e.runs)}" for e in self.entries]
        lines.append(f"best={self.best.name}")
        return "\n".join(lines) + "\n"

    def as_dict(self) -> dict:
        return {e.name: e.mean_seconds for e in self.entries}


def cuda_timer(fn) -> float:
    """Device seconds of one call of fn(), CUDA events on the current stream."""
    import torch
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) * 1e-3


def benchmark_candidate(fn, m: int = DEFAULT_M, timer=cuda_timer) -> float:
    """Mean duration over the last m of 2m+1 runs (autoselect.py:90-99)."""
    if m < 1:
        raise ValueError("m must be >= 1")
    runs = [timer(fn) for _ in range(2 * m + 1)]
    return float(statistics.fmean(runs[-m:]))


def benchmark_interleaved(candidates: dict, m: int = DEFAULT_M, timer=cuda_timer) -> BenchReport:
    """2m+1 rounds, one run of every candidate per round in the given order
    (autoselect.py:102-115); each candidate's figure is the mean of its own
    last m runs.  `candidates` maps name -> zero-argument callable."""
    if m < 1:
        raise ValueError("m must be >= 1")
    if not candidates:
        raise ValueError("no candidates")
    runs = {name: [] for name in candidates}
    for _ in range(2 * m + 1):
        for name, fn in candidates.items():
            runs[name].append(timer(fn))
    return BenchReport([BenchEntry(n, float(statistics.fmean(r[-m:])), r) for n, r in runs.items()])


@contextmanager
def plan_env(**knobs):
    """Temporarily set plan knobs the C ABI reads per call (PSN_TEAMS_FWD,
    PSN_TEAMS_BWD, PSN_LAG_FWD, PSN_LAG_BWD, PSN_STAGES, PSN_FORCE_GENERIC)."""
    old = {k: os.environ.get(k) for k in knobs}
    try:
        for k, v in knobs.items():
            os.environ[k] = str(v)
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def plan_variant(fn, **knobs):
    """A candidate: fn run under the given plan knobs."""
    def run():
        with plan_env(**knobs):
            fn()
    return run

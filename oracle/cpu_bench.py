"""CPU baseline timing of the oracle (the reference algorithm restated in
numpy) — TEST / BASELINE INFRASTRUCTURE ONLY, used by bench.py's
``cpu_baseline`` and ``--impl reference`` legs.

Runs SpikingLayer TRAIN forward + backward (the hot path) on a bounded sample
of the benchmark workload with every host core: channels are independent in
the PSN forward and backward (reference engines.py:132 acts per channel, and
every reduction is per channel), so splitting the channel axis across worker
processes computes exactly the reference's result, just in parallel.

Two figures (SURVEY.md section 8(d) "CPU path timing"):

* all host cores: the FULL workload (every channel, every batch row), channels
  split across one worker process per core;
* one core: a single process on a channel subset of the full workload, scaled
  per channel (every channel costs the same: same T, B, k, d), so the 1-core
  figure needs no multi-second run.

Prints one JSON line: {"value": Gsteps·ch/s (all cores), "one_core": {...}, ...}.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import platform
import time

import numpy as np

_X = None
_DY = None
_ARGS = None


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _work(sl):
    from oracle import psn_oracle as O
    lo, hi = sl
    k, d = _ARGS
    x = _X[:, :, lo:hi]
    dy = _DY[:, :, lo:hi]
    p = O.init_layer(hi - lo, k, d, weight_init="uniform", rng=np.random.default_rng(lo + 1))
    p.quantized = True
    out, cache, dx, dW, dg, db = O.train_step(p, x, dy)
    return float(dW.sum())


def single_core(T: int, B: int, C: int, k: int, d: int, csub: int, steps: int) -> dict:
    """One process, one thread: `csub` channels of the full [T, B, C] workload."""
    global _X, _DY, _ARGS
    csub = max(1, min(csub, C))
    rng = np.random.default_rng(0)
    _X = rng.standard_normal((T, B, csub)).astype(np.float32)
    _DY = rng.standard_normal((T, B, csub)).astype(np.float32)
    _ARGS = (k, d)
    _work((0, csub))  # warm-up (page faults, imports)
    times = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        _work((0, csub))
        times.append(time.perf_counter() - t0)
    sec = float(np.median(times)) * C / csub  # per full-width step
    return {"value": T * B * C / sec / 1e9, "unit": "Gsteps·ch/s", "seconds_per_step": sec, "cores": 1,
            "sample": f"T={T},B={B},k={k},d={d} fp32 TRAIN fwd+bwd on {csub} of {C} channels in one "
                      f"process (one thread), time scaled x{C / csub:g} to the full width"}


def run(T: int, B: int, C: int, k: int, d: int, steps: int, warmup: int, cores: int | None) -> dict:
    global _X, _DY, _ARGS
    cores = cores or os.cpu_count() or 1
    cores = max(1, min(cores, C))
    rng = np.random.default_rng(0)
    _X = rng.standard_normal((T, B, C)).astype(np.float32)
    _DY = rng.standard_normal((T, B, C)).astype(np.float32)
    _ARGS = (k, d)
    edges = np.linspace(0, C, cores + 1).astype(int)
    slices = [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(len(slices)) as pool:
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_work, slices)
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
    sec = float(np.median(times))
    return {"value": T * B * C / sec / 1e9, "unit": "Gsteps·ch/s", "seconds_per_step": sec,
            "cores": len(slices), "cpu_model": _cpu_model(), "host_cpus": os.cpu_count(),
            "steps": steps, "warmup": warmup,
            "sample": f"T={T},B={B},C={C},k={k},d={d} fp32 TRAIN fwd+bwd, channels split over "
                      f"{len(slices)} processes (exact: channels are independent)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=1024)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--C", type=int, default=512)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--d", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cores", type=int, default=0)
    ap.add_argument("--one-core-channels", type=int, default=16,
                    help="channels of the 1-core sample (0: skip the 1-core figure)")
    a = ap.parse_args()
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    res = run(a.T, a.B, a.C, a.k, a.d, a.steps, a.warmup, a.cores or None)
    if a.one_core_channels > 0:
        res["one_core"] = single_core(a.T, a.B, a.C, a.k, a.d, a.one_core_channels, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

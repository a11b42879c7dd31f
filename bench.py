"""Benchmark of the mul-free channel-wise PSN hot path (BASELINE.json metric):
SpikingLayer TRAIN forward + surrogate-gradient backward at T=1024, B=64,
C=512 (order 4, dilation 1, fp32 I/O, quantized, batch-stat BN fusion).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One process per GPU (torchrun for N>1, NCCL): each rank runs the layer on its
own batch of B=64 (weak scaling) and the per-channel parameter gradients are
all-reduced every step (DDP semantics).  Prints ONE JSON line on rank 0.

value   : Gsteps·ch/s = ranks * T*B*C / device time per step (max over ranks),
          inputs resident in HBM, CUDA events on the launch stream.
e2e     : the same metric through the public module API (SpikingLayer
          autograd) with x, dy in pinned host memory copied H2D inside the
          timed region and the gradients read back D2H every step.
roofline: algorithmic HBM bytes (20 B/elem fp32: fwd reads x, writes s; bwd
          reads x, dy, writes dx) of the dominant launch group over its
          CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
--impl reference: the reference algorithm (numpy oracle, every host core,
          channels split across processes) on a bounded sample.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "neuron fwd+bwd Gsteps·ch/s at T=1024,B=64,C=512; % HBM roofline; 1/2/4/8 GPU"
UNIT = "Gsteps·ch/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler running during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_baseline(args, steps=3, warmup=1, sample_B=8):
    """The oracle on every host core, bounded sample (subprocess: fork-safe)."""
    cmd = [sys.executable, "-m", "oracle.cpu_bench", "--T", str(args.T), "--B", str(sample_B), "--C",
           str(args.C), "--k", str(args.k), "--d", str(args.d), "--steps", str(steps), "--warmup", str(warmup)]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, env={**os.environ, "OMP_NUM_THREADS": "1"})
    if r.returncode != 0:
        return {"value": None, "error": r.stderr.strip()[-400:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def run_reference(args, rank: int, world: int):
    """--impl reference: the reference algorithm on the host cores, rank 0 only."""
    if rank != 0:
        return
    # every step is one bounded sample (B=8 of the workload, ~40 ms on 16 cores),
    # so the full --steps K --warmup W run stays within seconds to a minute
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    res = cpu_baseline(args, steps=steps, warmup=warmup)
    v = res.get("value")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": (res.get("seconds_per_step") or 0) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) x, dy; uniform(±k^-1/2) W",
        "config": {"workload": f"SpikingLayer TRAIN fwd+bwd T={args.T},B={args.B},C={args.C},k={args.k},"
                               f"d={args.d} fp32 quantized (bounded sample B=8)",
                   "parallelism": "host cores, channel split"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": res.get("cores"), "kind": "port",
                         "sample": res.get("sample"), "cpu_model": res.get("cpu_model")},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--T", type=int, default=1024)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--C", type=int, default=512)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--d", type=int, default=1)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time direct C-ABI calls instead of CUDA-graph replay")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2501_14490_b200 as P
    from paper_2501_14490_b200 import _lib as L

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    T, B, C, k, d = args.T, args.B, args.C, args.k, args.d
    dt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    esize = 4 if dt == torch.float32 else 2
    nel = T * B * C
    lib = L.lib()
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn((T, B, C), generator=g, device=dev).to(dt)
    dy = torch.randn((T, B, C), generator=g, device=dev).to(dt)
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(1), device=dev)
    flags = L.PSN_QUANTIZED | L.PSN_USE_BATCH_STATS
    desc = L.make_desc(x.shape, k, d, dt, flags=flags)
    ws = L.workspace(desc, dev)
    out = torch.empty_like(x)
    dx = torch.empty_like(x)
    fold = torch.empty((C, L.PSN_FOLD_HDR + 2 * k), dtype=torch.float64, device=dev)
    grads = torch.empty(C * k + 2 * C, dtype=torch.float64, device=dev)  # one flat DDP bucket
    dW, dgam, dbet = grads[:C * k], grads[C * k:C * k + C], grads[C * k + C:]
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    W, gam, bet, rm, rv = layer.W.detach(), layer.gamma.detach(), layer.beta.detach(), layer.running_mean, layer.running_var

    plan_f, plan_b = L.plan_info(desc, False), L.plan_info(desc, True)

    def fwd(s=None):
        L.check(lib.psn_forward_train(ctypes.byref(desc), x.data_ptr(), W.data_ptr(), gam.data_ptr(),
                                      bet.data_ptr(), rm.data_ptr(), rv.data_ptr(), out.data_ptr(),
                                      fold.data_ptr(), ws.data_ptr(), sp if s is None else s))

    def bwd(s=None):
        L.check(lib.psn_backward(ctypes.byref(desc), x.data_ptr(), dy.data_ptr(), W.data_ptr(), gam.data_ptr(),
                                 fold.data_ptr(), dx.data_ptr(), dW.data_ptr(), dgam.data_ptr(), dbet.data_ptr(),
                                 ws.data_ptr(), sp if s is None else s))

    # The timed step replays one CUDA graph per direction (the workspace clear
    # plus the persistent kernel), captured from the same C-ABI calls: this
    # removes the per-call launch and ramp-up gap of the cooperative launch
    # (~10 us fwd / ~5 us bwd when called directly).
    # --no-graph times the direct calls instead.
    if not args.no_graph:
        fwd(); bwd()
        torch.cuda.synchronize()
        g_f, g_b, g_s = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_f):
            fwd(torch.cuda.current_stream().cuda_stream)
        with torch.cuda.graph(g_b):
            bwd(torch.cuda.current_stream().cuda_stream)
        with torch.cuda.graph(g_s):  # the whole step in one graph: no gap between the two launches
            fwd(torch.cuda.current_stream().cuda_stream)
            bwd(torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        run_f, run_b, run_s = g_f.replay, g_b.replay, g_s.replay
    else:
        run_f, run_b = fwd, bwd

        def run_s():
            fwd()
            bwd()

    def step():
        run_s()
        if world > 1:
            dist.all_reduce(grads)

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    K = args.steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        ev[0].record(stream)
        for i in range(K):
            run_s()
            if world > 1:
                dist.all_reduce(grads)
            ev[i + 1].record(stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    step_ms = ev[0].elapsed_time(ev[K]) / K
    # per-launch times for the roofline: the same K steps again, one direction per event pair
    evd = [torch.cuda.Event(enable_timing=True) for _ in range(3 * K)]
    for i in range(K):
        evd[3 * i].record(stream)
        run_f()
        evd[3 * i + 1].record(stream)
        run_b()
        evd[3 * i + 2].record(stream)
    torch.cuda.synchronize()
    fwd_ms = [evd[3 * i].elapsed_time(evd[3 * i + 1]) for i in range(K)]
    bwd_ms = [evd[3 * i + 1].elapsed_time(evd[3 * i + 2]) for i in range(K)]
    t_local = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms = float(t_local.item())
    value = world * nel / (ms * 1e-3) / 1e9

    hbm, peak_src = _peaks()
    f_ms, b_ms = statistics.mean(fwd_ms), statistics.mean(bwd_ms)
    fwd_bytes, bwd_bytes = 2 * esize * nel, 3 * esize * nel
    fname = "psn_stream_kernel<fwd>" if plan_f.get("streamed") else "psn_forward_train (3 generic kernels)"
    bname = "psn_stream_kernel<bwd>" if plan_b.get("streamed") else "psn_backward (3 generic kernels)"
    groups = {fname: (fwd_bytes, f_ms), bname: (bwd_bytes, b_ms)}
    dom_name, (dom_bytes, dom_ms) = max(groups.items(), key=lambda kv: kv[1][1])
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None  # dram read+write bytes per launch of the dominant kernel, from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        key = next((kk for kk in tr if (("1>" in kk) == ("bwd" in dom_name)) and f"<{k}, {d}, float" in kk), None)
        if key is not None and args.dtype == "f32" and (T, B, C) == (1024, 64, 512):
            traffic = tr[key]["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        traffic = None
    step_achieved = (5 * esize * nel) / ((f_ms + b_ms) * 1e-3) / 1e9

    # ---- e2e through the public module API with host buffers -----------------
    e2e = None
    if not args.no_e2e:
        xh = torch.empty((T, B, C), dtype=dt, pin_memory=True)
        dyh = torch.empty((T, B, C), dtype=dt, pin_memory=True)
        xh.copy_(x.cpu())
        dyh.copy_(dy.cpu())
        gh = torch.empty(C * k + 2 * C, dtype=torch.float64, pin_memory=True)
        xd = torch.empty_like(x)
        dyd = torch.empty_like(dy)

        def e2e_step():
            xd.copy_(xh, non_blocking=True)
            dyd.copy_(dyh, non_blocking=True)
            xi = xd.requires_grad_(True)
            layer.zero_grad(set_to_none=True)
            layer(xi, P.Mode.TRAIN).backward(dyd)
            flat = torch.cat([layer.W.grad.flatten(), layer.gamma.grad, layer.beta.grad])
            if world > 1:
                dist.all_reduce(flat)
            gh.copy_(flat, non_blocking=True)
            xd.requires_grad_(False)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        ke = max(3, min(K, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / ke
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        e2e = {"value": world * nel / (ems * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": 2 * esize * nel, "d2h_bytes_per_step": 8 * (C * k + 2 * C),
               "api": "paper_2501_14490_b200.SpikingLayer autograd, pinned host x/dy"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)
        if cpu.get("value") is not None:
            cpu = {"value": cpu["value"], "unit": UNIT, "cores": cpu["cores"], "kind": "port",
                   "sample": cpu["sample"], "cpu_model": cpu.get("cpu_model")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic N(0,1) x and dy, uniform(±k^-1/2) W, gamma=1, beta=-1",
            "config": {"workload": f"SpikingLayer TRAIN fwd+bwd, quantized, batch-stat BN fusion, "
                                   f"T={T},B={B},C={C},k={k},d={d}, {args.dtype} I/O (BASELINE configs[4] "
                                   f"at the metric shape)",
                       "T": T, "B_per_gpu": B, "C": C, "k": k, "d": d, "parallelism": f"dp{world}",
                       "launch": "direct C-ABI calls" if args.no_graph else
                                 "CUDA-graph replay of the C-ABI calls (one graph per direction)",
                       "l2": "inputs larger than L2 (x, dy each %.0f MB > 126 MB L2)" % (nel * esize / 1e6)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "kernel": dom_name,
                         "algorithmic_bytes_per_launch": dom_bytes, "launch_ms": dom_ms,
                         "peak_source": peak_src},
            "step_roofline": {"achieved": step_achieved, "frac": step_achieved / hbm,
                              "bytes_per_step": 5 * esize * nel, "fwd_ms": f_ms, "bwd_ms": b_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": K * (plan_f["launches"] + plan_b["launches"]),
            "plan": {"forward": plan_f, "backward": plan_b},
            "clocks": clk.summary(),
            "wall_s_timed": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

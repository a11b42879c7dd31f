"""Benchmark of the mul-free channel-wise PSN hot path (BASELINE.json metric):
SpikingLayer TRAIN forward + surrogate-gradient backward at T=1024, B=64,
C=512 (order 4, dilation 1, fp32 I/O, quantized, batch-stat BN fusion).

    python bench.py [--gpus N --steps K --warmup W] [--scaling strong|weak] [--impl reference]

One process per GPU, NCCL.  `--gpus N` with N > 1
relaunches itself under torch.distributed.run when it is not already running
under it (and exits non-zero when WORLD_SIZE disagrees with N).  Prints ONE
JSON line on rank 0.

value   : Gsteps·ch/s of the whole job = T*B*C / device time per step (max over
          ranks), inputs resident in HBM, CUDA events on the launch stream.
          Default `--scaling strong`: the global batch B=64 is split across the
          ranks (ddp.shard_bounds, B=8 per GPU at N=8), as BASELINE.md section 2
          defines the 1/2/4/8-GPU metric.  N>1 also reports the weak-scaling
          figure (B=64 per rank) under "weak".  Every step all-reduces the
          per-channel gradients through ddp.GradBucket (NCCL).
e2e     : the same metric through the public module API (SpikingLayer autograd)
          from pinned host memory: x and dy are copied H2D and the spikes, dx
          and the gradient bucket D2H every step (copy streams overlap the
          previous / next step's compute).
roofline: algorithmic HBM bytes (20 B/elem fp32: fwd reads x, writes s; bwd
          reads x, dy, writes dx) of the dominant launch over its CUDA-event
          duration, against MEASURED_PEAKS.json hbm_gbs.
--impl reference: the reference algorithm (the numpy oracle, pinned bit-exact to
          the reference by tests/golden) on every host core, FULL workload,
          channels split across processes; rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
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


_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
period = float(sys.argv[2])
print("ready", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
while True:
    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    print(time.time(), mhz, r, flush=True)
    time.sleep(period)
"""


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler around the timed region, in its
    own process (a sampling thread would wait for the GIL while the benchmark
    thread launches and synchronises; one NVML clock query takes ~0.1-0.5 ms).
    Samples carry wall-clock stamps; the summary uses those taken inside the
    timed region, and the sampler runs until one sample lands after it."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.0002):
        self.index, self.period = index, period_s
        self.max_mhz = None
        self.proc = None
        self.ok = False
        self.lines = []
        self.t0 = self.t1 = None

    def _reader(self):
        for line in self.proc.stdout:
            self.lines.append(line)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.index), str(self.period)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline().split()
            if first and first[0] == "ready":
                self.max_mhz = int(first[1])
                self.ok = True
                self.rt = threading.Thread(target=self._reader, daemon=True)
                self.rt.start()
        except Exception:
            self.ok = False
        self.t0 = time.time()
        return self

    def _parsed(self):
        out = []
        for line in list(self.lines):
            parts = line.split()
            if len(parts) == 3:
                try:
                    out.append((float(parts[0]), int(parts[1]), int(parts[2])))
                except ValueError:
                    pass
        return out

    def __exit__(self, *a):
        self.t1 = time.time()
        if self.proc is None:
            return
        if self.ok:  # keep sampling until one sample is stamped after the region (<= 0.5 s)
            deadline = time.time() + 0.5
            while time.time() < deadline and not any(t >= self.t1 for t, _, _ in self._parsed()):
                time.sleep(0.001)
        self.proc.terminate()  # the sampler process this object started (exact PID)
        try:
            self.proc.wait(timeout=10)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            self.proc.wait()
        if self.ok:
            self.rt.join(timeout=5)

    def summary(self):
        s = self._parsed() if self.ok else []
        inside = [x for x in s if self.t0 <= x[0] <= self.t1]
        use = inside or [min(s, key=lambda x: abs(x[0] - self.t1))] if s else []
        reasons = set()
        for _, _, r in use:
            for bit, name in self.REASONS.items():
                if r & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(m for _, m, _ in use) if use else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(inside),
                "samples_total": len(s), "region_ms": round((self.t1 - self.t0) * 1e3, 2)}


# --------------------------------------------------------------------------
# launch plumbing
# --------------------------------------------------------------------------
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_if_needed(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: run N ranks under torch.distributed.run.
    Returns the child's exit code, or None when this process is already a rank."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus and args.gpus != 1:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
            return 2
        return None
    if args.gpus <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def batch_shard(B: int, rank: int, world: int, scaling: str) -> tuple[int, int]:
    """(rows on this rank, global batch): strong scaling splits the global batch
    B across the ranks (ddp.shard_bounds); weak scaling gives every rank B rows."""
    from paper_2501_14490_b200 import ddp
    if scaling == "weak":
        return B, B * world
    a, b = ddp.shard_bounds(B, rank, world)
    return b - a, B


# --------------------------------------------------------------------------
# CPU legs (the oracle; only here and in --impl reference)
# --------------------------------------------------------------------------
def cpu_baseline(args, steps=2, warmup=1, one_core_channels=16):
    """The oracle on every host core on the full workload + a 1-core figure
    (subprocess: fork-safe, outside any timed region)."""
    cmd = [sys.executable, "-m", "oracle.cpu_bench", "--T", str(args.T), "--B", str(args.B), "--C",
           str(args.C), "--k", str(args.k), "--d", str(args.d), "--steps", str(steps), "--warmup", str(warmup),
           "--one-core-channels", str(one_core_channels)]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, env={**os.environ, "OMP_NUM_THREADS": "1"})
    if r.returncode != 0:
        return {"value": None, "error": r.stderr.strip()[-400:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def _cpu_line(res):
    one = res.get("one_core") or {}
    return {"value": res.get("value"), "unit": UNIT, "cores": res.get("cores"), "kind": "port",
            "sample": res.get("sample"), "cpu_model": res.get("cpu_model"), "host_cpus": res.get("host_cpus"),
            "one_core": {"value": one.get("value"), "cores": 1, "sample": one.get("sample")} if one else None}


def run_reference(args, rank: int, world: int):
    """--impl reference: the reference algorithm on the host cores, rank 0 only.
    Each step is the full T*B*C workload (all channels, all batch rows), split
    by channel across one process per core."""
    if rank != 0:
        return
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    res = cpu_baseline(args, steps=steps, warmup=warmup, one_core_channels=8)
    v = res.get("value")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": (res.get("seconds_per_step") or 0) * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) x, dy; uniform(±k^-1/2) W",
        "config": {"workload": f"SpikingLayer TRAIN fwd+bwd T={args.T},B={args.B},C={args.C},k={args.k},"
                               f"d={args.d} fp32 quantized (full workload every step)",
                   "T": args.T, "B": args.B, "C": args.C, "k": args.k, "d": args.d,
                   "parallelism": "host cores, channel split", "same_config": True},
        "cpu_baseline": _cpu_line(res),
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if v is None:
        line["error"] = res.get("error")
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
class Workload:
    """One rank's share of the neuron layer step, driven through the C ABI:
    spikes/dx and a GradBucket whose views receive dW, dgamma, dbeta."""

    def __init__(self, P, L, dev, shape, k, d, dt, seed, use_graph, extra_flags=0):
        import numpy as np
        import torch
        from paper_2501_14490_b200 import ddp
        self.torch, self.L = torch, L
        C = shape[2]
        self.nel = 1
        for s_ in shape:
            self.nel *= s_
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.x = torch.randn(shape, generator=g, device=dev).to(dt)
        self.dy = torch.randn(shape, generator=g, device=dev).to(dt)
        cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
        self.layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(1), device=dev)
        flags = L.PSN_QUANTIZED | L.PSN_USE_BATCH_STATS | extra_flags
        self.desc = L.make_desc(self.x.shape, k, d, dt, flags=flags)
        self.ws = L.workspace(self.desc, dev)
        self.out = torch.empty_like(self.x)
        self.dx = torch.empty_like(self.x)
        self.fold = torch.empty((C, L.fold_stride(k)), dtype=torch.float64, device=dev)
        lay = self.layer
        self.bucket = ddp.GradBucket([lay.W, lay.gamma, lay.beta])
        self.dW, self.dgam, self.dbet = self.bucket.views()
        self.plan_f, self.plan_b = L.plan_info(self.desc, False), L.plan_info(self.desc, True)
        self.stream = torch.cuda.current_stream(dev)
        self.lib = L.lib()
        if use_graph:
            # one CUDA graph per direction and one for the whole step, captured
            # from the same C-ABI calls (removes the per-call launch / ramp gap
            # of the cooperative kernels)
            self.fwd(); self.bwd()
            torch.cuda.synchronize()
            gf, gb, gs = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(gf):
                self.fwd(torch.cuda.current_stream().cuda_stream)
            with torch.cuda.graph(gb):
                self.bwd(torch.cuda.current_stream().cuda_stream)
            with torch.cuda.graph(gs):
                self.fwd(torch.cuda.current_stream().cuda_stream)
                self.bwd(torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            self._graphs = (gf, gb, gs)
            self.run_f, self.run_b, self.run_s = gf.replay, gb.replay, gs.replay
        else:
            self.run_f, self.run_b = self.fwd, self.bwd

            def run_s():
                self.fwd()
                self.bwd()
            self.run_s = run_s

    def fwd(self, s=None):
        lay, L = self.layer, self.L
        L.check(self.lib.psn_forward_train(
            ctypes.byref(self.desc), self.x.data_ptr(), lay.W.data_ptr(), lay.gamma.data_ptr(),
            lay.beta.data_ptr(), lay.running_mean.data_ptr(), lay.running_var.data_ptr(), self.out.data_ptr(),
            self.fold.data_ptr(), self.ws.data_ptr(), self.stream.cuda_stream if s is None else s))

    def bwd(self, s=None):
        lay, L = self.layer, self.L
        L.check(self.lib.psn_backward(
            ctypes.byref(self.desc), self.x.data_ptr(), self.dy.data_ptr(), lay.W.data_ptr(),
            lay.gamma.data_ptr(), self.fold.data_ptr(), self.dx.data_ptr(), self.dW.data_ptr(),
            self.dgam.data_ptr(), self.dbet.data_ptr(), self.ws.data_ptr(),
            self.stream.cuda_stream if s is None else s))

    def step(self, world):
        self.run_s()
        if world > 1:
            self.bucket.reduce_()

    def time_steps(self, K, warmup, world, dist):
        torch = self.torch
        for _ in range(warmup):
            self.step(world)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(self.stream)
        for _ in range(K):
            self.step(world)
        ev[1].record(self.stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / K

    def time_directions(self, K):
        torch = self.torch
        evd = [torch.cuda.Event(enable_timing=True) for _ in range(3 * K)]
        for i in range(K):
            evd[3 * i].record(self.stream)
            self.run_f()
            evd[3 * i + 1].record(self.stream)
            self.run_b()
            evd[3 * i + 2].record(self.stream)
        torch.cuda.synchronize()
        f = [evd[3 * i].elapsed_time(evd[3 * i + 1]) for i in range(K)]
        b = [evd[3 * i + 1].elapsed_time(evd[3 * i + 2]) for i in range(K)]
        return statistics.mean(f), statistics.mean(b)


SUITE = [
    # (name, shape [T, B, C, *spatial], k, d, dtype): BASELINE.json configs, SURVEY.md section 8(d) inputs
    ("cfg1_T250_B32_C128_k4_d1", (250, 32, 128), 4, 1, "f32"),
    ("cfg1_T250_B32_C128_k4_d2", (250, 32, 128), 4, 2, "f32"),
    ("cfg1_T250_B32_C128_k4_d3", (250, 32, 128), 4, 3, "f32"),
    ("shard8_T1024_B8_C512_k4_d1", (1024, 8, 512), 4, 1, "f32"),
    ("seqcifar_T32_B128_C128x32_k16", (32, 128, 128, 32), 16, 1, "f32"),
    ("seqcifar_fc_T32_B128_C256_k16", (32, 128, 256), 16, 1, "f32"),
    ("dvslip_T30_B32_C64x22x22_k2_bf16", (30, 32, 64, 22, 22), 2, 1, "bf16"),
    ("dvslip_T30_B32_C512x3x3_k2_bf16", (30, 32, 512, 3, 3), 2, 2, "bf16"),
    ("sweep_T1024_k4_bf16", (1024, 64, 512), 4, 1, "bf16"),
    ("sweep_T1024_k8_d3", (1024, 64, 512), 8, 3, "f32"),
    ("sweep_T1024_k16_d3", (1024, 64, 512), 16, 3, "f32"),
    ("sweep_T4096_k4", (4096, 64, 512), 4, 1, "f32"),
    ("sweep_T16384_k4", (16384, 64, 512), 4, 1, "f32"),
]


def run_suite(P, L, dev, hbm, m=3):
    """Every BASELINE config on one GPU, timed with the 2m+1 / last-m protocol
    (paper_2501_14490_b200.protocol): per neuron layer shape fwd+bwd through
    the C ABI (CUDA-graph replay), and the SHD-shaped 3-layer full training
    step (Linear 700->128 and 128->128, PSN layers k and sawtooth d, readout,
    CE, Adam) through the module API."""
    import numpy as np
    import torch
    from paper_2501_14490_b200 import protocol
    from paper_2501_14490_b200.net import Adam, GraphedTrainStep, build_task_net
    out = {}
    for name, shape, k, d, dts in SUITE:
        dt = torch.float32 if dts == "f32" else torch.bfloat16
        try:
            wl = Workload(P, L, dev, shape, k, d, dt, 99, True)
            sec = protocol.benchmark_candidate(wl.run_s, m=m)
            es = 4 if dts == "f32" else 2
            out[name] = {"shape": list(shape), "k": k, "d": d, "dtype": dts, "ms": sec * 1e3,
                         "gsteps_ch_per_s": wl.nel / sec / 1e9,
                         "hbm_frac": 5 * es * wl.nel / sec / 1e9 / hbm,
                         "streamed": [wl.plan_f.get("streamed"), wl.plan_b.get("streamed")]}
            del wl
        except Exception as e:  # a config that cannot run is reported, not fatal
            out[name] = {"error": str(e)[:200]}
        torch.cuda.empty_cache()
    # SURVEY.md section 8(f) rank 1, the mul-free inference path at the metric
    # shape: SpikingLayer EVAL (running statistics folded, pow2 taps, one
    # spike kernel: reads x, writes spikes, 8 B/elem f32) and the quantized
    # file's ShiftLayer (psn_shift_spike_forward: the engine's ldexp arithmetic,
    # bit-exact to the reference, and the threshold in one pass)
    try:
        import numpy as np
        T, B, C = 1024, 64, 512
        g = torch.Generator(device=dev).manual_seed(7)
        xe = torch.randn((T, B, C), generator=g, device=dev)
        lay = P.SpikingLayer(P.NeuronConfig(channels=C, order=4, dilation=1, quantized=True),
                             weight_init="uniform", rng=np.random.default_rng(1), device=dev)
        lay.eval()

        def graphed(fn):  # one CUDA graph per call, like the TRAIN workload's replay
            fn()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                fn()
            return gr.replay
        sec = protocol.benchmark_candidate(graphed(lambda: lay(xe, P.Mode.EVAL)), m=m)
        out["eval_T1024_B64_C512_k4"] = {"ms": sec * 1e3, "gsteps_ch_per_s": T * B * C / sec / 1e9,
                                         "hbm_frac": 8 * T * B * C / sec / 1e9 / hbm,
                                         "what": "SpikingLayer EVAL (psn_forward_eval: fold + one spike kernel), "
                                                 "f32, CUDA-graph replay"}
        sw, bias = lay.quantized_snapshot()
        sl = P.ShiftLayer(sw, bias, 1)
        sec = protocol.benchmark_candidate(graphed(lambda: sl(xe, P.Mode.EVAL)), m=m)
        out["shift_eval_T1024_B64_C512_k4"] = {"ms": sec * 1e3, "gsteps_ch_per_s": T * B * C / sec / 1e9,
                                               "what": "ShiftLayer (quantized model file): psn_shift_spike_forward "
                                                       "(reference ldexp arithmetic and threshold in one pass), "
                                                       "CUDA-graph replay"}
        del xe, lay, sl
    except Exception as e:
        out["eval_T1024_B64_C512_k4"] = {"error": str(e)[:200]}
    torch.cuda.empty_cache()
    for korder in (2, 4):
        T, B, IN, H = 250, 128, 700, 128
        net = build_task_net(channels=H, num_layers=3, order=korder, classes=20, seed=0, in_features=IN,
                             device=dev)
        g = torch.Generator(device=dev).manual_seed(5)
        x = (torch.rand((T, B, IN), generator=g, device=dev) < 0.05).to(torch.float32)
        y = torch.randint(0, 20, (B,), generator=g, device=dev)
        opt = Adam(net.parameters_list(), 1e-3)

        def step():
            net.train_step_grads_async(x, y)
            opt.step()
        sec_eager = protocol.benchmark_candidate(step, m=m)
        graphed = GraphedTrainStep(net, opt, x, y)
        sec = protocol.benchmark_candidate(graphed, m=m)
        out[f"shd_train_step_T250_B128_in700_h128_k{korder}"] = {
            "ms": sec * 1e3, "ms_eager": sec_eager * 1e3, "samples_per_s": B / sec,
            "neuron_gsteps_ch_per_s": 3 * T * B * H / sec / 1e9,
            "what": "3 x (Linear + PSN layer, sawtooth d=1,2,3) + readout + CE + Adam, f32 activations; "
                    "one CUDA graph per step (GraphedTrainStep); ms_eager = the same step launched eagerly"}
        del net, opt, graphed
    return out


def max_over_ranks(v, world, dist, dev):
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_e2e(P, wl, world, dist, K):
    """The step through SpikingLayer autograd from pinned host memory: x, dy
    H2D and spikes, dx, gradient bucket D2H every step.  Three streams (H2D,
    compute, D2H) with two device slots, so step i's copies overlap step i+1's
    input copy and step i-1's result copy, as a data loader would."""
    import torch
    lay, x, dy = wl.layer, wl.x, wl.dy
    comp = wl.stream
    s_in, s_out = torch.cuda.Stream(x.device), torch.cuda.Stream(x.device)
    xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    dyh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    xh.copy_(x.cpu())
    dyh.copy_(dy.cpu())
    outh = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for _ in range(2)]
    dxh = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for _ in range(2)]
    gh = [torch.empty(wl.bucket.flat.shape, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    xd = [torch.empty_like(x) for _ in range(2)]
    dyd = [torch.empty_like(dy) for _ in range(2)]
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]

    def one(i):
        sl = i & 1
        with torch.cuda.stream(s_in):
            if used[sl]:
                s_in.wait_event(comp_done[sl])  # the slot's previous step consumed its inputs
            xd[sl].copy_(xh, non_blocking=True)
            dyd[sl].copy_(dyh, non_blocking=True)
            h2d_done[sl].record(s_in)
        comp.wait_event(h2d_done[sl])
        if used[sl]:
            comp.wait_event(d2h_done[sl])  # host result buffers of this slot are free again
        xi = xd[sl].requires_grad_(True)
        for p in (lay.W, lay.gamma, lay.beta):
            p.grad = None
        out = lay(xi, P.Mode.TRAIN)
        out.backward(dyd[sl])
        wl.bucket.pack()
        if world > 1:
            wl.bucket.reduce_()
        dx = xi.grad
        xi.grad = None
        xd[sl].requires_grad_(False)
        comp_done[sl].record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(comp_done[sl])
            out.record_stream(s_out)
            dx.record_stream(s_out)
            outh[sl].copy_(out, non_blocking=True)
            dxh[sl].copy_(dx, non_blocking=True)
            gh[sl].copy_(wl.bucket.flat, non_blocking=True)
            d2h_done[sl].record(s_out)
        used[sl] = True

    for i in range(2):
        one(i)
    torch.cuda.synchronize()
    ke = max(3, min(K, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    s_in.wait_stream(comp)
    for i in range(ke):
        one(i)
    comp.wait_stream(s_in)
    comp.wait_stream(s_out)
    e1.record(comp)
    torch.cuda.synchronize()
    ems = max_over_ranks(e0.elapsed_time(e1) / ke, world, dist, x.device)
    esize = x.element_size()
    return {"ms_per_step": ems, "h2d_bytes_per_step": 2 * esize * wl.nel,
            "d2h_bytes_per_step": 2 * esize * wl.nel + 8 * wl.bucket.flat.numel(),
            "api": "paper_2501_14490_b200.SpikingLayer autograd; pinned host x/dy in, spikes/dx/grads out; "
                   "H2D, compute and D2H on three streams (two device slots)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: global batch --B split across ranks (default); weak: --B per rank")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: multi-rank tests on one device)")
    ap.add_argument("--T", type=int, default=1024)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--C", type=int, default=512)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--d", type=int, default=1)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-weak", action="store_true", help="N>1: skip the extra weak-scaling measurement")
    ap.add_argument("--no-suite", action="store_true", help="skip the per-config suite (BASELINE configs 1-5)")
    ap.add_argument("--no-graph", action="store_true", help="time direct C-ABI calls instead of CUDA-graph replay")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rc = relaunch_if_needed(args)
    if rc is not None:
        sys.exit(rc)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2501_14490_b200 as P
    from paper_2501_14490_b200 import _lib as L

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local % max(ndev, 1))
    torch.cuda.set_device(dev)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    T, C, k, d = args.T, args.C, args.k, args.d
    dt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    esize = 4 if dt == torch.float32 else 2
    Bl, Bg = batch_shard(args.B, rank, world, args.scaling)
    wl = Workload(P, L, dev, (T, Bl, C), k, d, dt, 1234 + rank, not args.no_graph)
    K = args.steps

    with ClockSampler(dev.index) as clk:
        t0 = time.perf_counter()
        step_ms = wl.time_steps(K, args.warmup, world, dist)
        wall = time.perf_counter() - t0
    ms = max_over_ranks(step_ms, world, dist, dev)
    value = T * Bg * C / (ms * 1e-3) / 1e9
    f_ms, b_ms = wl.time_directions(K)

    weak = None
    if world > 1 and not args.no_weak:
        other = "weak" if args.scaling == "strong" else "strong"
        Bl2, Bg2 = batch_shard(args.B, rank, world, other)
        wl2 = Workload(P, L, dev, (T, Bl2, C), k, d, dt, 4321 + rank, not args.no_graph)
        ms2 = max_over_ranks(wl2.time_steps(K, args.warmup, world, dist), world, dist, dev)
        weak = {"scaling": other, "value": T * Bg2 * C / (ms2 * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms2,
                "B_per_gpu": Bl2, "global_batch": Bg2}
        del wl2

    hbm, peak_src = _peaks()
    nel = wl.nel
    fwd_bytes, bwd_bytes = 2 * esize * nel, 3 * esize * nel
    fname = "psn_stream_kernel<fwd>" if wl.plan_f.get("streamed") else "psn_forward_train (3 generic kernels)"
    bname = "psn_stream_kernel<bwd>" if wl.plan_b.get("streamed") else "psn_backward (3 generic kernels)"
    groups = {fname: (fwd_bytes, f_ms), bname: (bwd_bytes, b_ms)}
    dom_name, (dom_bytes, dom_ms) = max(groups.items(), key=lambda kv: kv[1][1])
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None  # dram read+write bytes per launch of the dominant kernel, from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        def _tmpl(kk):  # "psn_stream_kernel<K, D, float, BWD, SP>" -> ["K", "D", "float", "BWD", "SP"]
            return [t.strip() for t in kk[kk.index("<") + 1:kk.rindex(">")].split(",")]
        key = next((kk for kk in tr if _tmpl(kk)[:4] == [str(k), str(d), "float", "1" if "bwd" in dom_name else "0"]),
                   None)
        if key is not None and args.dtype == "f32" and (T, Bl, C) == (1024, 64, 512):
            traffic = tr[key]["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        traffic = None
    step_achieved = (5 * esize * nel) / ((f_ms + b_ms) * 1e-3) / 1e9

    e2e = None
    if not args.no_e2e:
        e = run_e2e(P, wl, world, dist, K)
        e2e = {"value": T * Bg * C / (e["ms_per_step"] * 1e-3) / 1e9, "unit": UNIT, **e}

    suite = None
    if rank == 0 and world == 1 and not args.no_suite:
        suite = run_suite(P, L, dev, _peaks()[0])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = cpu_baseline(args)
        cpu = _cpu_line(res) if res.get("value") is not None else res

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic N(0,1) x and dy, uniform(±k^-1/2) W, gamma=1, beta=-1",
            "config": {"workload": f"SpikingLayer TRAIN fwd+bwd, quantized, batch-stat BN fusion, "
                                   f"T={T},B={Bg},C={C},k={k},d={d}, {args.dtype} I/O (BASELINE metric shape; "
                                   f"{args.scaling} scaling, B={Bl} on rank 0)",
                       "T": T, "global_batch": Bg, "B_per_gpu": Bl, "C": C, "k": k, "d": d,
                       "parallelism": f"dp{world}",
                       "launch": "direct C-ABI calls" if args.no_graph else
                                 "CUDA-graph replay of the C-ABI calls (fwd+bwd in one graph)",
                       "l2": "inputs larger than L2 (x, dy each %.0f MB vs 126 MB L2)" % (nel * esize / 1e6)
                             if nel * esize > 126e6 else
                             "per-rank inputs (%.0f MB) fit L2; consecutive steps reuse them" % (nel * esize / 1e6)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "kernel": dom_name,
                         "algorithmic_bytes_per_launch": dom_bytes, "launch_ms": dom_ms,
                         "peak_source": peak_src},
            "step_roofline": {"achieved": step_achieved, "frac": step_achieved / hbm,
                              "bytes_per_step": 5 * esize * nel, "fwd_ms": f_ms, "bwd_ms": b_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            # kernels of this repo per timed step (the streamed plans' workspace
            # memset is a driver memset node, not counted)
            "gpu_launches": K * sum(pl["launches"] - (1 if pl.get("streamed") else 0)
                                    for pl in (wl.plan_f, wl.plan_b)),
            "plan": {"forward": wl.plan_f, "backward": wl.plan_b},
            "clocks": clk.summary(),
            "wall_s_timed": wall,
        }
        if weak is not None:
            line["weak"] = weak
        if suite is not None:
            line["suite"] = suite
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""How many clock samples bench.py's sampler gets over a short busy region."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
x = torch.randn(1 << 26, device="cuda")
for region_ms in (5, 20, 100):
    with bench.ClockSampler(0) as clk:
        t0 = time.perf_counter()
        while (time.perf_counter() - t0) * 1e3 < region_ms:
            x.mul_(1.0000001)
            torch.cuda.synchronize()
    print(region_ms, "ms region:", clk.summary())

# the bench's own timed region (CUDA-graph replays of the metric step)
import paper_2501_14490_b200 as P
from paper_2501_14490_b200 import _lib as L
wl = bench.Workload(P, L, torch.device("cuda:0"), (1024, 64, 512), 4, 1, torch.float32, 1, True)
for K in (20, 200):
    with bench.ClockSampler(0) as clk:
        t0 = time.perf_counter()
        ms = wl.time_steps(K, 5, 1, None)
        wall = time.perf_counter() - t0
    print(f"K={K}: {ms:.4f} ms/step, wall {wall * 1e3:.1f} ms:", clk.summary())

"""bf16 k=16 on the generic kernels (ring vs register-prefetch A/B helper)."""
import torch, bench, paper_2501_14490_b200 as P
from paper_2501_14490_b200 import _lib as L, protocol
dev = torch.device("cuda:0")
for shape, k, d in (((1024, 64, 512), 16, 3), ((1024, 64, 512), 16, 1), ((1024, 64, 512), 12, 2), ((32, 128, 128, 32), 16, 1)):
    wl = bench.Workload(P, L, dev, shape, k, d, torch.bfloat16, 5, True)
    sec = protocol.benchmark_candidate(wl.run_s, m=2)
    print(shape, k, d, "bf16", round(sec * 1e3, 4), flush=True)
    del wl

"""SURVEY.md section 8(d) input (5), the long sweep: T in {1k, 2k, 4k, 8k, 16k},
k in {4, 8, 16}, d in {1, 2, 3}, f32 and bf16, B=64, C=512, one GPU; fwd+bwd
per step through the C ABI (CUDA-graph replay, 2m+1/last-m protocol), with
the kernel family the planner picked and the fraction of the HBM roofline
(20 B/elem f32, 10 B/elem bf16).

    PYTHONPATH=. python scripts/sweep_long.py > profiles/r2_sweep_long.txt
"""
import torch

import bench
import paper_2501_14490_b200 as P
from paper_2501_14490_b200 import _lib as L
from paper_2501_14490_b200 import protocol

dev = torch.device("cuda:0")
hbm = bench._peaks()[0]
print(f"# B=64, C=512; ms per fwd+bwd step; HBM peak {hbm} GB/s; family = streamed (S) / generic (G)")
print(f"{'T':>6s} {'k':>3s} {'d':>2s} {'dtype':>5s} {'family':>6s} {'ms':>9s} {'Gsteps.ch/s':>12s} {'frac':>6s}")
for dts in ("f32", "bf16"):
    dt = torch.float32 if dts == "f32" else torch.bfloat16
    es = 4 if dts == "f32" else 2
    for T in (1024, 2048, 4096, 8192, 16384):
        for k in (4, 8, 16):
            for d in (1, 2, 3):
                wl = bench.Workload(P, L, dev, (T, 64, 512), k, d, dt, 5, True)
                sec = protocol.benchmark_candidate(wl.run_s, m=2)
                fam = "S" if wl.plan_b.get("streamed") else "G"
                print(f"{T:6d} {k:3d} {d:2d} {dts:>5s} {fam:>6s} {sec * 1e3:9.4f} {wl.nel / sec / 1e9:12.1f} "
                      f"{5 * es * wl.nel / sec / 1e9 / hbm:6.3f}", flush=True)
                del wl
                torch.cuda.empty_cache()

"""Time a subset of bench.py's per-config suite (neuron-layer fwd+bwd through
the C ABI, CUDA-graph replay, 2m+1/last-m protocol).

    PYTHONPATH=. python scripts/gen_suite.py [name-substring ...]
"""
import json
import sys

import torch

import bench
import paper_2501_14490_b200 as P
from paper_2501_14490_b200 import _lib as L
from paper_2501_14490_b200 import protocol

keys = sys.argv[1:] or [""]
dev = torch.device("cuda:0")
for name, shape, k, d, dts in bench.SUITE:
    if not any(s in name for s in keys):
        continue
    dt = torch.float32 if dts == "f32" else torch.bfloat16
    wl = bench.Workload(P, L, dev, shape, k, d, dt, 99, True)
    sec = protocol.benchmark_candidate(wl.run_s, m=3)
    print(json.dumps({"name": name, "ms": round(sec * 1e3, 4), "gsteps_ch_per_s": round(wl.nel / sec / 1e9, 2),
                      "streamed": [wl.plan_f.get("streamed"), wl.plan_b.get("streamed")]}), flush=True)
    del wl
    torch.cuda.empty_cache()

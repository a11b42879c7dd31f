"""Time a subset of bench.py's per-config suite (neuron-layer fwd+bwd through
the C ABI, CUDA-graph replay, 2m+1/last-m protocol), plus extra shapes.

    PYTHONPATH=. python scripts/gen_suite.py [--generic] [--extra] [name-substring ...]

--generic sets the PSN_GENERIC descriptor flag (three-launch kernels);
--extra adds the routing-calibration shapes below.
"""
import json
import sys

import torch

import bench
import paper_2501_14490_b200 as P
from paper_2501_14490_b200 import _lib as L
from paper_2501_14490_b200 import protocol

EXTRA = [
    ("metric_k4_d1", (1024, 64, 512), 4, 1, "f32"), ("metric_k4_d2", (1024, 64, 512), 4, 2, "f32"),
    ("metric_k4_d3", (1024, 64, 512), 4, 3, "f32"), ("metric_k2_d1", (1024, 64, 512), 2, 1, "f32"),
    ("metric_k8_d1", (1024, 64, 512), 8, 1, "f32"), ("metric_k8_d2", (1024, 64, 512), 8, 2, "f32"),
    ("metric_k6_d3", (1024, 64, 512), 6, 3, "f32"), ("shard8_k4_d3", (1024, 8, 512), 4, 3, "f32"),
    ("T512_B16_C256_k4_d1", (512, 16, 256), 4, 1, "f32"), ("T1024_B16_C512_k4_d1", (1024, 16, 512), 4, 1, "f32"),
    ("T1024_B32_C512_k4_d1", (1024, 32, 512), 4, 1, "f32"),
]
args = sys.argv[1:]
generic = "--generic" in args
extra = "--extra" in args
keys = [a for a in args if not a.startswith("--")] or [""]
dev = torch.device("cuda:0")
for name, shape, k, d, dts in bench.SUITE + (EXTRA if extra else []):
    if not any(s in name for s in keys):
        continue
    dt = torch.float32 if dts == "f32" else torch.bfloat16
    wl = bench.Workload(P, L, dev, shape, k, d, dt, 99, True, extra_flags=L.PSN_GENERIC if generic else 0)
    sec = protocol.benchmark_candidate(wl.run_s, m=3)
    print(json.dumps({"name": name, "generic": generic, "ms": round(sec * 1e3, 4),
                      "gsteps_ch_per_s": round(wl.nel / sec / 1e9, 2),
                      "streamed": [wl.plan_f.get("streamed"), wl.plan_b.get("streamed")]}), flush=True)
    del wl
    torch.cuda.empty_cache()

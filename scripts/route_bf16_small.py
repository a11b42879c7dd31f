import torch, bench, paper_2501_14490_b200 as P
from paper_2501_14490_b200 import _lib as L, protocol
dev = torch.device("cuda:0")
for shape in ((250, 32, 128), (512, 16, 128), (30, 32, 64, 7, 7)):
    for d in (1, 3):
        for fl, nm in ((L.PSN_STREAM, "stream"), (L.PSN_GENERIC, "generic")):
            wl = bench.Workload(P, L, dev, shape, 4 if len(shape) == 3 else 2, d, torch.bfloat16, 5, True, extra_flags=fl)
            sec = protocol.benchmark_candidate(wl.run_s, m=3)
            print(shape, d, nm, round(sec * 1e3, 4), wl.plan_b.get("streamed"), flush=True)
            del wl

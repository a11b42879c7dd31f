import torch, bench, paper_2501_14490_b200 as P
from paper_2501_14490_b200 import _lib as L, protocol
dev = torch.device("cuda:0")
for T in (1024, 4096):
    for fl, nm in ((L.PSN_STREAM, "stream"), (L.PSN_GENERIC, "generic")):
        for dt in (torch.bfloat16, torch.float32):
            wl = bench.Workload(P, L, dev, (T, 64, 512), 8, 3, dt, 5, True, extra_flags=fl)
            sec = protocol.benchmark_candidate(wl.run_s, m=2)
            print(T, nm, dt, round(sec * 1e3, 4), wl.plan_b.get("streamed"), flush=True)
            del wl

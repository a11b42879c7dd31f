"""Microbenchmark: synapse backward pieces at the SHD shape (32000 rows)."""
import torch


def t(fn, n=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


R = 32000
for IN in (700, 128):
    x = (torch.rand(R, IN, device="cuda") < 0.05).float()
    g = torch.randn(R, 128, device="cuda")
    ones = torch.ones(1, R, device="cuda")
    print(IN, "db g.sum(0)", round(t(lambda: g.sum(0)), 1))
    print(IN, "db ones@g", round(t(lambda: ones @ g), 1))
    print(IN, "db view-sum", round(t(lambda: g.view(250, 128, 128).sum(1).sum(0)), 1))
    print(IN, "dW g.t()@x", round(t(lambda: g.t() @ x), 1))
    for S in (8, 16, 32, 64):
        gs, xs = g.view(S, R // S, 128), x.view(S, R // S, IN)
        print(IN, f"dW bmm S={S}", round(t(lambda: torch.bmm(gs.transpose(1, 2), xs).sum(0)), 1))
    gx = torch.cat([g, torch.ones(R, 1, device="cuda")], 1)
    print(IN, "dW+db fused [g|1]^T x", round(t(lambda: gx.t() @ x), 1))

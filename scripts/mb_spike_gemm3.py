"""Microbenchmark: spike-input synapse forward as ONE bf16 GEMM against the
three bf16 parts of W stacked ([W_hi; W_mid; W_lo], N = 3*out) plus the sum of
the three column blocks, vs the f32 SIMT GEMM (SHD shape)."""
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
    W = torch.randn(128, IN, device="cuda")
    hi = W.bfloat16(); r = W - hi.float(); mid = r.bfloat16(); lo = (r - mid.float()).bfloat16()
    W3 = torch.cat([hi, mid, lo], 0)  # [384, IN]
    xb = x.bfloat16()
    print(IN, "f32 linear", round(t(lambda: torch.nn.functional.linear(x, W)), 1))
    print(IN, "x->bf16", round(t(lambda: x.bfloat16()), 1))
    print(IN, "bf16 GEMM N=384 out f32", round(t(lambda: torch.mm(xb, W3.t(), out_dtype=torch.float32)), 1))
    y3 = torch.mm(xb, W3.t(), out_dtype=torch.float32)
    print(IN, "sum blocks", round(t(lambda: y3.view(R, 3, 128).sum(1)), 1))
    y = y3.view(R, 3, 128).sum(1)
    ref = x.double() @ W.double().t()
    print(IN, "max rel err", float(((y.double() - ref).abs() / ref.abs().clamp(min=1)).max()),
          "f32:", float(((torch.nn.functional.linear(x, W).double() - ref).abs() / ref.abs().clamp(min=1)).max()))

"""Microbenchmark: f32 F.linear vs the split-bf16 spike synapse (SHD layer-1 shape)."""
import torch, torch.nn.functional as F
from paper_2501_14490_b200.net import LinearLayer, _split3_bf16
from paper_2501_14490_b200.layer import Mode
import numpy as np

def t(fn, n=20):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3

for IN in (700, 128):
    x = (torch.rand(250, 128, IN, device="cuda") < 0.05).float()
    W = torch.randn(128, IN, device="cuda", dtype=torch.float64)
    W32 = W.float()
    xb = x.reshape(-1, IN).bfloat16()
    parts = _split3_bf16(W32)
    g = torch.randn(250 * 128, 128, device="cuda")
    print(IN, "F.linear f32 us", t(lambda: F.linear(x, W32)))
    print(IN, "x->bf16 us", t(lambda: x.reshape(-1, IN).bfloat16()))
    print(IN, "mm bf16 out f32 us", t(lambda: torch.mm(xb, parts[0].t(), out_dtype=torch.float32)))
    print(IN, "mm bf16 out bf16 us", t(lambda: torch.mm(xb, parts[0].t())))
    print(IN, "mm f32 dW us", t(lambda: torch.mm(g.t(), x.reshape(-1, IN))))
    print(IN, "mm bf16 dW us", t(lambda: torch.mm(g.bfloat16().t(), xb, out_dtype=torch.float32)))
    print(IN, "split g us", t(lambda: _split3_bf16(g)))
    print(IN, "dx f32 us", t(lambda: torch.mm(g, W32)))
    lin = LinearLayer(IN, 128, rng=np.random.default_rng(0), device="cuda", spike_input=True)
    xr = x.clone().requires_grad_(IN == 128)
    def fb(spike):
        lin.spike_input = spike
        y = lin(xr, Mode.TRAIN); y.backward(g.reshape(250, 128, 128))
    print(IN, "layer fwd+bwd spike us", t(lambda: fb(True)), "plain us", t(lambda: fb(False)))

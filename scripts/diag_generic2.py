"""Streamed vs generic method on identical inputs at the metric shape: where do
the results differ (diagnostic)."""
import numpy as np
import torch

import paper_2501_14490_b200 as P

for d in (1, 2, 3):
    rng = np.random.default_rng(203)
    shape = (1024, 64, 512)
    x_np = rng.standard_normal(shape).astype(np.float32)
    dy_np = rng.standard_normal(shape).astype(np.float32)
    res = {}
    for method in ("stream", "generic"):
        cfg = P.NeuronConfig(channels=512, order=4, dilation=d, quantized=True)
        layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(204), device="cuda")
        layer.configure(P.layer.LayerMethod(method))
        x = torch.tensor(x_np, device="cuda", requires_grad=True)
        out = layer(x, P.Mode.TRAIN)
        out.backward(torch.tensor(dy_np, device="cuda"))
        st = {k: v.cpu().numpy() for k, v in layer.last_state().items()}
        res[method] = dict(out=out.detach().cpu().numpy(), dx=x.grad.cpu().numpy(), dW=layer.W.grad.cpu().numpy(),
                           dg=layer.gamma.grad.cpu().numpy(), db=layer.beta.grad.cpu().numpy(), **st)
    a, b = res["stream"], res["generic"]
    print(f"d={d}: spikes differ {int((a['out'] != b['out']).sum())}")
    for k in ("mu", "s", "a", "b_f", "w_q", "dx", "dW", "dg", "db"):
        diff = np.abs(a[k].astype(np.float64) - b[k])
        scale = np.maximum(np.abs(a[k]), 1.0)
        i = np.unravel_index(np.argmax(diff / scale), diff.shape)
        print(f"   {k:4s} max scaled diff {float((diff / scale).max()):.3e} at {i} (stream {a[k][i]!r} generic {b[k][i]!r})")

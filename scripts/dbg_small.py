import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2501_14490_b200 as P
for (T,N,C,k,d) in [(64,4,32,2,1),(300,20,64,2,1)]:
    for bwd in (False, True):
        cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
        layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(1), device="cuda")
        x = torch.randn((T,N,C), device="cuda", requires_grad=True)
        out = layer(x, P.Mode.TRAIN)
        torch.cuda.synchronize(); print("fwd ok", T,N,C,k,d, flush=True)
        if bwd:
            out.backward(torch.randn_like(out)); torch.cuda.synchronize(); print("bwd ok", flush=True)

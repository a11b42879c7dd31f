"""Quick bounded check of the fused kernels on a few shapes (run under `timeout`)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_14490_b200 as P
shapes = [((64, 4, 32), 4, 2), ((250, 32, 128), 4, 3), ((256, 16, 256), 4, 1), ((1024, 64, 512), 4, 1)]
for shp, k, d in shapes:
    t0 = time.time()
    cfg = P.NeuronConfig(channels=shp[2], order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(1), device="cuda")
    x = torch.randn(shp, device="cuda", requires_grad=True)
    out = layer(x, P.Mode.TRAIN)
    torch.cuda.synchronize()
    print("fwd ok", shp, round(time.time() - t0, 2), flush=True)
    out.backward(torch.randn(shp, device="cuda"))
    torch.cuda.synchronize()
    print("bwd ok", shp, round(time.time() - t0, 2), flush=True)

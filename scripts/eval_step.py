"""SpikingLayer EVAL at the metric shape (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_14490_b200 as P
x = torch.randn((1024, 64, 512), device="cuda")
lay = P.SpikingLayer(P.NeuronConfig(channels=512, order=4, dilation=1, quantized=True), weight_init="uniform",
                     rng=np.random.default_rng(1), device="cuda")
lay.eval()
for _ in range(5):
    lay(x, P.Mode.EVAL)
torch.cuda.synchronize()

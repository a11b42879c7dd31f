"""One small fwd+bwd (f32 and bf16) through the C ABI, for compute-sanitizer.

    python scripts/san_step.py T N C k d [method]   (method: auto | stream | generic)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_14490_b200 as P
T, N, C, k, d = (int(v) for v in sys.argv[1:6])
method = sys.argv[6] if len(sys.argv) > 6 else "auto"
for dt in (torch.float32, torch.bfloat16):
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(1), device="cuda")
    layer.configure(P.layer.LayerMethod(method))
    x = torch.randn((T, N, C), device="cuda").to(dt).requires_grad_(True)
    layer(x, P.Mode.TRAIN).backward(torch.randn((T, N, C), device="cuda").to(dt))
    torch.cuda.synchronize()
flags = 5 | {"auto": 0, "stream": P._lib.PSN_STREAM, "generic": P._lib.PSN_GENERIC}[method]
print("plan", P._lib.plan_info(P._lib.make_desc((T, N, C), k, d, torch.float32, flags=flags), True))

"""Parity diagnostic (GPU): max errors of the CUDA path vs the oracle for a
few shapes/dtypes, printed per output (bounded; run under gpurun)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_14490_b200 as P
from oracle import psn_oracle as O


def run(T, N, C, k, d, spatial=(), dtype=torch.float32, channels=(0, 1), seed=0):
    rng = np.random.default_rng(seed)
    shape = (T, N, C) + tuple(spatial)
    x_np = rng.standard_normal(shape).astype(np.float32)
    dy_np = rng.standard_normal(shape).astype(np.float32)
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(seed + 1), device="cuda")
    x = torch.tensor(x_np, device="cuda", dtype=dtype, requires_grad=True)
    out = layer(x, P.Mode.TRAIN)
    out.backward(torch.tensor(dy_np, device="cuda", dtype=dtype))
    sel = np.array(channels)
    xs = x.detach().float().cpu().numpy()[:, :, sel]
    dys = torch.tensor(dy_np, dtype=dtype).float().numpy()[:, :, sel]
    p = O.init_layer(len(sel), k, d, weight_init="uniform", rng=np.random.default_rng(seed + 1))
    p.W = layer.W.detach().cpu().numpy()[sel]
    ref_out, cache, dx, dW, dg, db = O.train_step(p, xs, dys)
    gdx = x.grad.float().cpu().numpy()[:, :, sel].astype(np.float64)
    e = np.abs(gdx - dx)
    i = np.unravel_index(np.argmax(e / (np.abs(dx) + 1e-3)), e.shape)
    got = out.detach().float().cpu().numpy()[:, :, sel]
    print(f"shape={shape} k={k} d={dtype} spk_mism={int((got != ref_out).sum())} "
          f"dx maxerr={e.max():.3e} maxrel={np.max(e / np.maximum(np.abs(dx), 1e-30)):.3e} at {i} ref={dx[i]:.4e} got={gdx[i]:.4e} "
          f"dW err={np.abs(layer.W.grad.cpu().numpy()[sel] - dW).max():.3e} mu err={np.abs(layer.last_state()['mu'].cpu().numpy()[sel]-cache.mu).max():.3e}",
          flush=True)


for spec in sys.argv[1:] or ["dvs"]:
    if spec == "dvs":
        run(30, 32, 64, 2, 2, (22, 22), torch.bfloat16, (0, 31, 63), 30)
        run(30, 32, 64, 2, 2, (22, 22), torch.float32, (0, 31, 63), 30)
        run(30, 32, 64, 2, 2, (), torch.bfloat16, (0, 31, 63), 30)
        os.environ["PSN_FORCE_GENERIC"] = "1"
        run(30, 32, 64, 2, 2, (), torch.bfloat16, (0, 31, 63), 30)
        run(256, 16, 128, 2, 1, (), torch.bfloat16, (0, 5), 5)
        del os.environ["PSN_FORCE_GENERIC"]

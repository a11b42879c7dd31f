"""GPU parity of the full training step around the neuron (SURVEY.md section
8(f) rank 2) and of quantized export (rank 3) against fixtures the reference
wrote (tests/golden/make_golden_net.py): SpikingNet.train_step_grads with the
reference's Adam, two steps; EVAL logits; SSNN1 files of the trained net."""

import os
import socket

import numpy as np
import pytest
import torch

from tests.parity import assert_close_scaled, assert_rel

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _z():
    return np.load(os.path.join(GOLDEN, "net_train.npz"))


def _net(dtype=torch.float64):
    from paper_2501_14490_b200.net import build_task_net
    T, N, IN, CH, CLASSES, ORDER, SEED = (int(v) for v in _z()["meta"])
    return build_task_net(channels=CH, num_layers=3, order=ORDER, classes=CLASSES, seed=SEED,
                          in_features=IN, device="cuda")


def _train_two_steps(net, dtype=torch.float64):
    from paper_2501_14490_b200.net import Adam
    z = _z()
    params = net.parameters_list()
    opt = Adam(params, float(z["lr"]))
    res = []
    for step in range(2):
        x = torch.tensor(z[f"s{step}_x"], device="cuda", dtype=dtype)
        y = torch.tensor(z[f"s{step}_y"], device="cuda")
        loss, acc = net.train_step_grads(x, y)
        grads = [p.grad.detach().cpu().numpy().copy() for p in params]
        stats = [(l.running_mean.cpu().numpy().copy(), l.running_var.cpu().numpy().copy())
                 for l in net.spiking_layers()]
        opt.step()
        res.append((loss, acc, grads, stats, [p.detach().cpu().numpy().copy() for p in params]))
    return res


def test_training_step_matches_reference_f64():
    """float64 carrier: the reference's TRAIN arithmetic (Linear, PSN layers on
    the generic f64 kernels, readout, CE, Adam), two steps."""
    z = _z()
    net = _net()
    for step, (loss, acc, grads, stats, after) in enumerate(_train_two_steps(net)):
        assert abs(loss - float(z[f"s{step}_loss"])) <= 1e-12 * max(1.0, abs(float(z[f"s{step}_loss"])))
        assert acc == float(z[f"s{step}_acc"])
        for i, g in enumerate(grads):
            assert_close_scaled(g, z[f"s{step}_grad_{i}"], 1e-9, f"step {step} grad {i}")
        for j, (rm, rv) in enumerate(stats):
            assert_rel(rm, z[f"s{step}_rm_{j}"], 1e-10, f"running_mean {j}")
            assert_rel(rv, z[f"s{step}_rv_{j}"], 1e-10, f"running_var {j}")
        for i, p in enumerate(after):
            assert_close_scaled(p, z[f"s{step}_after_{i}"], 1e-9, f"step {step} param {i}")


def test_eval_logits_and_predictions_match_reference():
    from paper_2501_14490_b200.layer import Mode
    z = _z()
    net = _net()
    _train_two_steps(net)
    xe = torch.tensor(z["eval_x"], device="cuda")
    logits = net(xe, Mode.EVAL).detach().double().cpu().numpy()
    assert_close_scaled(logits, z["eval_logits"], 1e-5, "eval logits (f32 deployment path)")
    assert np.array_equal(net.predict(xe).cpu().numpy(), z["eval_pred"])


def test_quantized_export_matches_reference_file():
    """quantized_snapshot (running stats folded, pow2-quantized on the GPU) of
    the trained net gives the reference's sign / exponent bytes; the fused
    f32 biases agree to an f32 ulp."""
    from paper_2501_14490_b200 import modelio
    net = _net()
    _train_two_steps(net)
    got = modelio.model_bytes(net, quantize=True)
    want = open(os.path.join(GOLDEN, "ssnn1_quantized.bin"), "rb").read()
    assert len(got) == len(want)
    gnet, _ = modelio.model_from_bytes(got, device="cpu")
    wnet, _ = modelio.model_from_bytes(want, device="cpu")
    for a, b in zip(gnet.layers, wnet.layers):
        assert type(a) is type(b)
        if hasattr(a, "sw"):
            assert torch.equal(a.sw.sign, b.sw.sign) and torch.equal(a.sw.exponent, b.sw.exponent)
            assert a.dilation == b.dilation
            assert_close_scaled(a.bias.numpy(), b.bias.numpy(), 2 ** -22, "fused bias")
        else:
            assert_close_scaled(a.W.detach().numpy(), b.W.detach().numpy(), 2 ** -22, "weights")


def test_quantized_model_inference_matches_reference():
    """The reference's quantized file reloads as ShiftLayers; the EVAL logits of
    the mul-free network equal the reference's."""
    from paper_2501_14490_b200 import modelio
    from paper_2501_14490_b200.layer import Mode
    z = _z()
    qnet, meta = modelio.load_model(os.path.join(GOLDEN, "ssnn1_quantized.bin"), device="cuda")
    assert meta["quantized"]
    logits = qnet(torch.tensor(z["eval_x"], device="cuda"), Mode.EVAL).detach().double().cpu().numpy()
    want = np.load(os.path.join(GOLDEN, "net_quantized_eval.npz"))["q_eval_logits"]
    assert_close_scaled(logits, want, 1e-5, "quantized eval logits")


def test_readout_kernels_against_reference_recurrence():
    """psn_readout_reduce / _expand vs the reference's sequential leaky
    accumulator (network.py:413-436) on random data, f32 / f64 / bf16 carriers."""
    from paper_2501_14490_b200.net import ReadoutLayer
    rng = np.random.default_rng(3)
    for dt in (torch.float64, torch.float32, torch.bfloat16):
        T, N, C, K = 37, 5, 11, 3
        x = torch.tensor(rng.standard_normal((T, N, C)), device="cuda").to(dt)
        ro = ReadoutLayer(C, K, tau=2.5, rng=np.random.default_rng(1), device="cuda")
        xr = x.double().requires_grad_(True)
        logits = ro(x.detach().requires_grad_(True) if dt != torch.float64 else xr)
        xd = x.detach().double().cpu().numpy()
        W, b = ro.W.detach().cpu().numpy(), ro.b.detach().cpu().numpy()
        cur = np.einsum("tnc,oc->tno", xd, W) + b
        inv = 1.0 / ro.tau
        v = np.zeros_like(cur[0])
        for t in range(T):
            v = (1 - inv) * v + inv * cur[t]
        assert_close_scaled(logits.detach().cpu().numpy(), v, 1e-12, f"logits {dt}")
        g = rng.standard_normal((N, K))
        xin = x.detach().clone().requires_grad_(True)
        ro(xin).backward(torch.tensor(g, device="cuda"))
        gg = g.copy()
        dcur = np.empty((T, N, K))
        for t in range(T - 1, -1, -1):
            dcur[t] = inv * gg
            gg = (1 - inv) * gg
        dx = np.einsum("tno,oc->tnc", dcur, W)
        tol = {torch.float64: 1e-12, torch.float32: 1e-6, torch.bfloat16: 2 ** -8}[dt]
        assert_close_scaled(xin.grad.double().cpu().numpy(), dx, tol, f"dx {dt}")
        assert_close_scaled(ro.W.grad.cpu().numpy(), np.einsum("tno,tnc->oc", dcur, xd), 1e-12, f"dW {dt}")


@pytest.mark.parametrize("method", ["stream", "auto"])
def test_f32_network_trains(method):
    """The production setting: f32 activations through the PSN kernels (the
    streamed ones, and the planner's choice: the three generic launches at
    this small shape); the step runs, its loss tracks the f64 reference's, and
    training reduces the loss on a fixed batch."""
    import paper_2501_14490_b200 as P
    from paper_2501_14490_b200.net import Adam
    z = _z()
    net = _net()
    for layer in net.layers:
        if isinstance(layer, P.SpikingLayer):
            layer.configure(P.layer.LayerMethod(method))
    x = torch.tensor(z["s0_x"], device="cuda", dtype=torch.float32)
    y = torch.tensor(z["s0_y"], device="cuda")
    loss0, _ = net.train_step_grads(x, y)
    assert abs(loss0 - float(z["s0_loss"])) < 1e-3
    opt = Adam(net.parameters_list(), 1e-2)
    for _ in range(30):
        net.train_step_grads(x, y)
        opt.step()
    loss1, _ = net.train_step_grads(x, y)
    assert loss1 < loss0


def test_graphed_train_step_equals_eager():
    """The captured step (forward, CE, backward, Adam in one CUDA graph) gives
    the eager step's losses and parameters on the f32 streamed path (both run
    the capturable Adam, whose bias corrections come from the device)."""
    from paper_2501_14490_b200.net import Adam, GraphedTrainStep
    z = _z()
    x = torch.tensor(z["s0_x"], device="cuda", dtype=torch.float32)
    y = torch.tensor(z["s0_y"], device="cuda")
    nets, losses = [], []
    for graphed in (False, True):
        net = _net()
        opt = Adam(net.parameters_list(), 1e-2)
        opt.make_capturable()
        if graphed:
            step = GraphedTrainStep(net, opt, x, y, warmup=3)
            ls = [float(step()[0]) for _ in range(3)]
        else:
            ls = []
            for _ in range(6):
                loss, _ = net.train_step_grads_async(x, y)
                opt.step()
                ls.append(float(loss))
            ls = ls[3:]
        nets.append(net)
        losses.append(ls)
    assert losses[0] == losses[1]
    for a, b in zip(nets[0].parameters_list(), nets[1].parameters_list()):
        assert torch.equal(a, b)


def test_explicit_layer_backward_matches_autograd():
    """SpikingLayer.backward(dy) (the reference's layer-by-layer API) returns
    autograd's dx and accumulates the same parameter gradients."""
    import paper_2501_14490_b200 as P
    cfg = P.NeuronConfig(channels=64, order=4, dilation=2, quantized=True)
    a = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(2), device="cuda")
    b = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(2), device="cuda")
    x = torch.randn(200, 12, 64, device="cuda")
    dy = torch.randn(200, 12, 64, device="cuda")
    xa = x.clone().requires_grad_(True)
    a(xa, P.Mode.TRAIN).backward(dy)
    b(x, P.Mode.TRAIN)
    dx = b.backward(dy)
    assert torch.equal(dx, xa.grad)
    for pa, pb in zip(a.parameters_list(), b.parameters_list()):
        assert torch.equal(pa.grad, pb.grad)
    b.backward(dy)  # accumulates like the reference's +=
    assert torch.equal(b.W.grad, 2 * a.W.grad)
    assert [m.name for m in b.method_candidates()] == ["auto", "stream", "generic"]
    with pytest.raises(ValueError):
        b.configure(P.layer.LayerMethod("matmul"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ddp_worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2501_14490_b200 import ddp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = _z()
        net = _net()
        x = torch.tensor(z["s0_x"], device="cuda")
        y = torch.tensor(z["s0_y"], device="cuda")
        a, b = ddp.shard_bounds(x.shape[1], rank, world)
        net.train_step_grads(x[:, a:b].contiguous(), y[a:b])
        bucket = ddp.GradBucket(net.parameters_list())
        bucket.allreduce()
        out[rank] = [p.grad.cpu().numpy().copy() for p in net.parameters_list()]
    finally:
        dist.destroy_process_group()


def test_ddp_step_two_ranks_on_product_kernels():
    """World size 2 (gloo, both ranks on cuda:0): each rank runs the product
    kernels on its batch shard; the bucketed all-reduce gives the sum of the
    per-shard gradients a single process computes."""
    import torch.multiprocessing as mp
    from paper_2501_14490_b200 import ddp
    z = _z()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ddp_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    x = torch.tensor(z["s0_x"], device="cuda")
    y = torch.tensor(z["s0_y"], device="cuda")
    want = None
    for r in range(2):
        net = _net()
        a, b = ddp.shard_bounds(x.shape[1], r, 2)
        net.train_step_grads(x[:, a:b].contiguous(), y[a:b])
        g = [p.grad.cpu().numpy() for p in net.parameters_list()]
        want = g if want is None else [u + v for u, v in zip(want, g)]
    for r in range(2):
        for got, w in zip(out[r], want):
            np.testing.assert_allclose(got, w, rtol=1e-12, atol=1e-14)


def test_fused_adam_matches_the_reference_update():
    """psn_adam_step (all tensors in one launch) against a float64 numpy
    restatement of the reference's Adam (train.py:147-172; true division, as
    numpy does): bit-identical with host bias corrections, and within an ulp
    of the corrections with the device step count (device pow)."""
    from paper_2501_14490_b200.net import Adam
    rng = np.random.default_rng(3)
    b1, b2, lr, eps = 0.9, 0.999, 1e-2, 1e-8
    for capturable in (False, True):
        ref = [rng.standard_normal(n) for n in (5000, 17, 4096, 1)]
        ps = [torch.tensor(r, device="cuda") for r in ref]
        ms = [np.zeros_like(r) for r in ref]
        vs = [np.zeros_like(r) for r in ref]
        opt = Adam(ps, lr)
        if capturable:
            opt.make_capturable()
        for t in range(1, 4):
            grads = [rng.standard_normal(r.shape) for r in ref]
            for p, g in zip(ps, grads):
                p.grad = torch.tensor(g, device="cuda")
            opt.step()
            c1, c2 = 1 - b1 ** t, 1 - b2 ** t
            for i, g in enumerate(grads):
                ms[i] = ms[i] * b1 + (1 - b1) * g
                vs[i] = vs[i] * b2 + (1 - b2) * g * g
                ref[i] = ref[i] - lr * (ms[i] / c1) / (np.sqrt(vs[i] / c2) + eps)
            for p, r in zip(ps, ref):
                got = p.cpu().numpy()
                if capturable:
                    np.testing.assert_allclose(got, r, rtol=1e-14, atol=1e-16)
                else:
                    assert np.array_equal(got, r), (t, float(np.abs(got - r).max()))


def test_split_k_synapse_backward_matches_f64():
    """The f32 synapse's split-K weight gradient and GEMV bias gradient against
    the float64 products of the same f32 inputs (f32 accumulation over 32000
    rows: cuBLAS's single f32 GEMM is off by up to ~3e-5 of max(|ref|, 1)
    here too, scripts/diag_dw_f32.py)."""
    from paper_2501_14490_b200.layer import Mode
    from paper_2501_14490_b200.net import LinearLayer
    lin = LinearLayer(700, 128, rng=np.random.default_rng(4), device="cuda")
    x = (torch.rand(250, 128, 700, device="cuda") < 0.05).float().requires_grad_(True)
    y = lin(x, Mode.TRAIN)
    gy = torch.randn_like(y)
    y.backward(gy)
    xd, gd = x.detach().double(), gy.double()
    W32 = lin.W.detach().float().double()
    assert_close_scaled(lin.W.grad.cpu().numpy(), torch.einsum("tno,tni->oi", gd, xd).cpu().numpy(), 1e-4, "dW")
    assert_close_scaled(lin.b.grad.cpu().numpy(), gd.sum(dim=(0, 1)).cpu().numpy(), 1e-4, "db")
    assert_close_scaled(x.grad.double().cpu().numpy(), torch.einsum("tno,oi->tni", gd, W32).cpu().numpy(), 1e-5,
                        "dx")

"""GPU parity of SpikingLayer (CUDA path through the C ABI) against the
reference: golden fixtures produced by the reference itself, plus the oracle
at the benchmark's full sizes on channel subsets (channels are independent in
forward and backward, so a subset is an exact restatement of the full job)."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import psn_oracle as O
from tests.parity import assert_close_scaled, assert_rel, spikes_match_except_ties

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))
CASES = {c["name"]: c for c in MANIFEST["layer_cases"]}


def _P():
    import paper_2501_14490_b200 as P
    return P


def _layer_from_fixture(meta, z):
    P = _P()
    f = meta["flags"]
    kind, alpha = f.get("surrogate", ["arctan", 2.0])
    cfg = P.NeuronConfig(channels=meta["shape"][2], order=meta["k"], dilation=meta["d"],
                         weight_sharing=P.WeightSharing.SHARED if f.get("shared") else P.WeightSharing.CHANNEL_WISE,
                         quantized=f.get("quantized", True),
                         grad_mode=P.QuantGradMode.ROUND_STE if f.get("grad_mode") == "round_ste"
                         else P.QuantGradMode.WHOLE_STE)
    layer = P.SpikingLayer(cfg, surrogate=P.SurrogateConfig(P.SurrogateKind(kind), alpha),
                           fuse_from_batch_stats=f.get("fuse_from_batch_stats", True), device="cuda")
    layer.quantize_in_smooth_mode = bool(f.get("quantize_in_smooth_mode", False))
    with torch.no_grad():
        layer.W.copy_(torch.from_numpy(z["W"]))
        layer.gamma.copy_(torch.from_numpy(z["gamma"]))
        layer.beta.copy_(torch.from_numpy(z["beta"]))
        layer.running_mean.copy_(torch.from_numpy(z["running_mean_in"]))
        layer.running_var.copy_(torch.from_numpy(z["running_var_in"]))
    return layer


@pytest.mark.parametrize("method", ["stream", "generic"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_layer_matches_reference_fixture(name, method):
    P = _P()
    meta = CASES[name]
    z = np.load(os.path.join(GOLDEN, f"layer_{name}.npz"))
    layer = _layer_from_fixture(meta, z)
    layer.configure(P.layer.LayerMethod(method))
    smooth = meta["mode"] == "smooth"
    mode = P.Mode.SMOOTH if smooth else P.Mode.TRAIN
    f64 = meta["dtype"] == "float64"
    gtol = 1e-9 if f64 else 1e-5
    d = meta["d"]
    for step in range(2):
        pre = f"s{step}_"
        x = torch.tensor(z[pre + "x"], device="cuda", requires_grad=True)
        out = layer(x, mode)
        st = {k: v.cpu().numpy() for k, v in layer.last_state().items()}
        assert_rel(st["mu"], z[pre + "mu"], 1e-11, "mu")
        assert_rel(st["s"], z[pre + "s"], 1e-12, "s")
        assert_rel(st["a"], z[pre + "a"], 1e-12, "a")
        assert_close_scaled(st["b_f"], z[pre + "b_f"], 1e-12, "b_f")
        assert_rel(st["w_f"], z[pre + "w_f"], 1e-12, "w_f")
        if meta["flags"].get("quantized", True) and (not smooth or meta["flags"].get("quantize_in_smooth_mode")):
            assert np.array_equal(st["w_q"], z[pre + "w_q"]), "quantized weights differ"
        else:
            assert_rel(st["w_q"], z[pre + "w_q"], 1e-12, "w_q (float)")
        assert_rel(layer.running_mean.cpu().numpy(), z[pre + "running_mean"], 1e-10, "running_mean")
        assert_rel(layer.running_var.cpu().numpy(), z[pre + "running_var"], 1e-12, "running_var")
        got = out.detach().cpu().numpy()
        assert got.dtype == z[pre + "x"].dtype
        if smooth:
            assert_close_scaled(got, z[pre + "out"], 1e-12 if f64 else 1e-6, "smooth output")
        else:
            spikes_match_except_ties(got, z[pre + "out"], z[pre + "x"], z[pre + "w_q"], z[pre + "b_f"], d)
        layer.zero_grad(set_to_none=True)
        out.backward(torch.tensor(z[pre + "dy"], device="cuda"))
        assert_close_scaled(x.grad.cpu().numpy(), z[pre + "dx"], gtol, "dx")
        assert_close_scaled(layer.W.grad.cpu().numpy(), z[pre + "dW"], gtol, "dW")
        assert_close_scaled(layer.gamma.grad.cpu().numpy(), z[pre + "dgamma"], gtol, "dgamma")
        assert_close_scaled(layer.beta.grad.cpu().numpy(), z[pre + "dbeta"], gtol, "dbeta")
    # EVAL with the running statistics after the two steps (network.py:219-234)
    layer.eval()
    xe = torch.tensor(z["eval_x"], device="cuda")
    got = layer(xe).cpu().numpy()
    p = O.LayerParams(W=z["W"], gamma=z["gamma"], beta=z["beta"],
                      running_mean=layer.running_mean.cpu().numpy(),
                      running_var=layer.running_var.cpu().numpy(), d=d,
                      quantized=meta["flags"].get("quantized", True))
    w_f, b_f = O.fused_running(p)
    w = O.dequantize(*O.quantize_pow2(w_f)) if p.quantized else w_f.astype(np.float32).astype(np.float64)
    b = b_f.astype(np.float32).astype(np.float64)
    spikes_match_except_ties(got, z["eval_out"], z["eval_x"].astype(np.float32), w, b, d, "eval spikes")


def _oracle_subset_check(T, N, C, k, d, channels, dtype=torch.float32, seed=0, spatial=(), x_fn=None,
                         method="stream"):
    """Full-size GPU fwd+bwd; oracle on a channel subset (exact restatement:
    channels are independent in forward and backward).  `spatial` adds axes
    after C (rank 4/5, the reference's [T, N, C, H, W]); `x_fn(rng, shape)`
    replaces the N(0, 1) input draw."""
    P = _P()
    rng = np.random.default_rng(seed)
    shape = (T, N, C) + tuple(spatial)
    x_np = (x_fn(rng, shape) if x_fn is not None else rng.standard_normal(shape)).astype(np.float32)
    dy_np = rng.standard_normal(shape).astype(np.float32)
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(seed + 1), device="cuda")
    layer.configure(P.layer.LayerMethod(method))
    x = torch.tensor(x_np, device="cuda", dtype=dtype, requires_grad=True)
    out = layer(x, P.Mode.TRAIN)
    out.backward(torch.tensor(dy_np, device="cuda", dtype=dtype))
    torch.cuda.synchronize()
    sel = np.array(channels)
    xs = x.detach().float().cpu().numpy()[:, :, sel]
    dys = torch.tensor(dy_np, dtype=dtype).float().numpy()[:, :, sel]
    p = O.init_layer(len(sel), k, d, weight_init="uniform", rng=np.random.default_rng(seed + 1))
    p.W = layer.W.detach().cpu().numpy()[sel]
    ref_out, cache, dx, dW, dg, db = O.train_step(p, xs, dys)
    st = {kk: v.cpu().numpy()[sel] for kk, v in layer.last_state().items()}
    # mean: 1e-10 relative, or 1e-12 of the channel's spread when the mean is
    # near zero (any two summation orders of the reference's mean differ by
    # ~1e-16 * mean|h1|, so a relative bound alone is ill-conditioned there)
    mu_err = np.abs(st["mu"] - cache.mu)
    assert np.all(mu_err <= 1e-10 * np.abs(cache.mu) + 1e-12 * cache.s), f"mu: max err {mu_err.max():.3e}"
    assert_rel(st["a"], cache.a, 1e-12, "a")
    assert np.array_equal(st["w_q"], cache.w_q)
    got = out.detach().float().cpu().numpy()[:, :, sel]
    flips = spikes_match_except_ties(got, ref_out, xs, cache.w_q, cache.b_f, d)
    gdx = x.grad.float().cpu().numpy()[:, :, sel]
    if dtype == torch.float32:
        assert_close_scaled(gdx, dx, 1e-5, "dx")
    else:  # bf16 dx: the f32 result rounded to bf16 (half an ulp <= 2^-8 |dx|) + the f32 bound
        err = np.abs(gdx.astype(np.float64) - dx)
        bound = 2.0 ** -8 * np.abs(dx) + 1e-5 * np.maximum(np.abs(dx), 1.0)
        assert not (err > bound).any(), f"bf16 dx: {int((err > bound).sum())} outside; max err {err.max():.3e}"
    assert_close_scaled(layer.W.grad.cpu().numpy()[sel], dW, 1e-5, "dW")
    assert_close_scaled(layer.gamma.grad.cpu().numpy()[sel], dg, 1e-5, "dgamma")
    assert_close_scaled(layer.beta.grad.cpu().numpy()[sel], db, 1e-5, "dbeta")
    return flips


@pytest.mark.parametrize("d", [1, 2, 3])
def test_metric_config_parity_on_channel_subset(d):
    """T=1024, B=64, C=512, k=4 (BASELINE metric config), sawtooth d."""
    flips = _oracle_subset_check(1024, 64, 512, 4, d, channels=[0, 1, 77, 255, 256, 400, 510, 511], seed=d)
    assert flips <= 2


def test_routing_rule():
    """The planner's choice (PSN_STREAM / PSN_GENERIC unset): BASELINE config 1
    (1.0M elements) and k = 8, d = 3 on the generic kernels, the metric shape
    and the 8-GPU shard on the streamed ones; PSN_STREAM overrides."""
    from paper_2501_14490_b200 import _lib as L
    base = L.PSN_QUANTIZED | L.PSN_USE_BATCH_STATS
    for shape, k, d, dt, want in [((250, 32, 128), 4, 1, torch.float32, 0), ((1024, 64, 512), 8, 3, torch.float32, 0),
                                  ((1024, 64, 512), 4, 1, torch.float32, 1), ((1024, 8, 512), 4, 3, torch.float32, 1),
                                  ((1024, 64, 512), 6, 3, torch.float32, 1), ((1024, 64, 512), 8, 3, torch.bfloat16, 0),
                                  ((250, 32, 128), 4, 1, torch.bfloat16, 0)]:
        for bwd in (False, True):
            assert L.plan_info(L.make_desc(shape, k, d, dt, flags=base), bwd)["streamed"] == want, (shape, dt)
            assert L.plan_info(L.make_desc(shape, k, d, dt, flags=base | L.PSN_STREAM), bwd)["streamed"] == 1
            assert L.plan_info(L.make_desc(shape, k, d, dt, flags=base | L.PSN_GENERIC), bwd)["streamed"] == 0


@pytest.mark.parametrize("d", [1, 2, 3])
def test_metric_config_parity_generic_method(d):
    """The metric config through the generic three-launch kernels (descriptor
    flag PSN_GENERIC: the shared-memory-ring streaming loops and the
    materialised dh2 / h1 - mu backward)."""
    flips = _oracle_subset_check(1024, 64, 512, 4, d, channels=list(range(0, 512, 4)), seed=200 + d,
                                 method="generic")
    assert flips <= 4


@pytest.mark.parametrize("shape,k,d,dt,off", [
    ((250, 32, 128), 4, 1, torch.float32, 0.0),     # config 1
    ((300, 7, 45), 16, 3, torch.float32, 50.0),     # ragged tile (J % 4 != 0: scalar copies), offset mean
    ((64, 5, 12, 3, 3), 6, 2, torch.float32, 0.0),  # spatial, k > 4
    ((200, 9, 96), 8, 3, torch.bfloat16, 0.0),      # bf16: register prefetch
])
def test_generic_method_parity(shape, k, d, dt, off):
    T, N, C = shape[:3]
    flips = _oracle_subset_check(T, N, C, k, d, channels=list(range(C)), dtype=dt, seed=7, spatial=shape[3:],
                                 x_fn=lambda rng, sh: rng.standard_normal(sh) + off, method="generic")
    assert flips <= 4


@pytest.mark.parametrize("d", [1, 2, 3])
def test_metric_config_parity_all_channels(d):
    """The BASELINE metric config in full: T=1024, B=64, C=512, k=4, every
    channel checked against the oracle (~7 s of numpy per d)."""
    flips = _oracle_subset_check(1024, 64, 512, 4, d, channels=list(range(512)), seed=100 + d)
    assert flips <= 8


def test_long_sequence_parity_t16384():
    """Long-sequence sweep endpoint T=16384, B=64, C=512 (BASELINE configs[4]);
    oracle on a channel subset spread over the channel groups."""
    _oracle_subset_check(16384, 64, 512, 4, 1, channels=[0, 95, 300, 511], seed=16)


def test_offset_mean_inputs_stress_the_moments():
    """Inputs whose membrane mean is far from the (initial, zero) running mean:
    x + 50 (mean/std of h1 ~ 100) -- the one-pass moments must still give the
    reference's two-pass mean/var (neuron.py:185-191) to 1e-10."""
    _oracle_subset_check(1024, 64, 128, 4, 2, channels=list(range(128)), seed=50,
                         x_fn=lambda rng, shape: rng.standard_normal(shape) + 50.0)


def test_nonnegative_spike_inputs():
    """Spike-driven currents (non-negative, sparse): Bernoulli(0.05) events
    scaled by a positive synaptic weight, as a spiking layer's input sees."""
    _oracle_subset_check(1024, 64, 128, 4, 3, channels=list(range(128)), seed=51,
                         x_fn=lambda rng, shape: (rng.random(shape) < 0.05) * rng.uniform(0.5, 2.0, shape))


def test_seq_cifar_shape_k16_parity():
    """seq-CIFAR conv-stage neuron tensor [T=32, B=128, C=128, 32] at order 16
    (BASELINE configs[2]); oracle on a channel subset."""
    _oracle_subset_check(32, 128, 128, 16, 1, channels=[0, 63, 127], seed=32, spatial=(32,))


def test_dvs_lip_shape_bf16_parity():
    """DVS-Lip stage-1 neuron tensor [T=30, B=32, C=64, 22, 22], order 2, bf16
    I/O (BASELINE configs[3]); oracle on the bf16 inputs widened to f32."""
    _oracle_subset_check(30, 32, 64, 2, 2, channels=[0, 31, 63], dtype=torch.bfloat16, seed=30,
                         spatial=(22, 22))


@pytest.mark.parametrize("shape,k,d,dt", [
    ((64, 20, 40, 3, 3), 4, 3, torch.float32),    # Q = 9: 32 channels per group, 9 column tiles
    ((40, 16, 13, 12), 3, 2, torch.float32),      # Q = 12, C = 13: one partial group
    ((48, 18, 40, 12), 2, 1, torch.float32),      # Q = 12, C = 40: 2 groups, the last partial
    ((32, 24, 48, 32), 4, 1, torch.float32),      # Q = 32 (seq-CIFAR conv stage): 8 channels per group
    ((30, 32, 16, 22, 22), 2, 3, torch.bfloat16), # Q = 484 (DVS-Lip stage 1), bf16
])
def test_spatial_inputs_streamed_parity(shape, k, d, dt):
    """Spatial inputs [T, N, C, H(, W)] on the streamed kernels: channel groups
    span several 32-column tiles and the per-channel sums merge the column sums
    (segmented warp scan); every channel against the oracle."""
    from paper_2501_14490_b200 import _lib as L
    desc = L.make_desc(shape, k, d, dt, flags=L.PSN_QUANTIZED | L.PSN_USE_BATCH_STATS | L.PSN_STREAM)
    assert L.plan_info(desc, False)["streamed"] == 1 and L.plan_info(desc, True)["streamed"] == 1
    T, N, C = shape[:3]
    _oracle_subset_check(T, N, C, k, d, channels=list(range(C)), dtype=dt, seed=sum(shape) + k,
                         spatial=shape[3:], method="stream")


FLAG_CASES = [
    # name, (T, N, C), k, d, flags
    ("shared", (301, 23, 64), 3, 2, dict(shared=True)),
    ("round_ste", (257, 20, 64), 4, 1, dict(round_ste=True)),
    ("rational", (300, 16, 96), 4, 2, dict(surrogate="rational", alpha=10.0)),
    ("float_weights", (200, 18, 64), 5, 1, dict(quantized=False)),
    ("running_fusion", (250, 24, 64), 4, 3, dict(fuse_from_batch_stats=False)),
    ("k6d3", (333, 17, 32), 6, 3, {}),
    ("k7d2", (129, 40, 96), 7, 2, {}),
    ("k8d1", (100, 16, 64), 8, 1, {}),
    ("k8d3_T_lt_halo", (19, 16, 32), 8, 3, {}),
]


@pytest.mark.parametrize("method", ["stream", "generic"])
@pytest.mark.parametrize("name,shape,k,d,flags", FLAG_CASES, ids=[c[0] for c in FLAG_CASES])
def test_flag_matrix_two_steps(name, shape, k, d, flags, method):
    """The streamed and the generic kernels under every layer option the
    reference has (shared weights, ROUND_STE, rational surrogate, float
    weights, running-stat fusion), orders 3-8, T and N off the tile grid,
    random gamma / beta / running stats; two steps, so the second uses the
    running statistics the first updated."""
    P = _P()
    from paper_2501_14490_b200 import _lib as L
    T, N, C = shape
    rng = np.random.default_rng(sum(map(ord, name)))
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=flags.get("quantized", True),
                         weight_sharing=P.WeightSharing.SHARED if flags.get("shared") else P.WeightSharing.CHANNEL_WISE,
                         grad_mode=P.QuantGradMode.ROUND_STE if flags.get("round_ste") else P.QuantGradMode.WHOLE_STE)
    sur = P.SurrogateConfig(P.SurrogateKind(flags.get("surrogate", "arctan")), flags.get("alpha", 2.0))
    layer = P.SpikingLayer(cfg, surrogate=sur, weight_init="uniform", rng=np.random.default_rng(7), device="cuda",
                           fuse_from_batch_stats=flags.get("fuse_from_batch_stats", True))
    layer.configure(P.layer.LayerMethod(method))
    gamma, beta = rng.uniform(0.5, 1.5, C), rng.uniform(-1.5, 0.5, C)
    rm, rv = rng.normal(0.0, 0.3, C), rng.uniform(0.5, 2.0, C)
    with torch.no_grad():
        layer.gamma.copy_(torch.from_numpy(gamma))
        layer.beta.copy_(torch.from_numpy(beta))
        layer.running_mean.copy_(torch.from_numpy(rm))
        layer.running_var.copy_(torch.from_numpy(rv))
    desc = L.make_desc(shape, k, d, torch.float32, flags=layer._flags(P.Mode.TRAIN))
    want = 1 if method == "stream" else 0
    assert L.plan_info(desc, False)["streamed"] == want and L.plan_info(desc, True)["streamed"] == want
    p = O.init_layer(C, k, d, weight_init="uniform", rng=np.random.default_rng(7), shared=flags.get("shared", False),
                     quantized=flags.get("quantized", True), round_ste=flags.get("round_ste", False),
                     fuse_from_batch_stats=flags.get("fuse_from_batch_stats", True),
                     surrogate=flags.get("surrogate", "arctan"), alpha=flags.get("alpha", 2.0))
    p.W = layer.W.detach().cpu().numpy().copy()
    p.gamma, p.beta, p.running_mean, p.running_var = gamma.copy(), beta.copy(), rm.copy(), rv.copy()
    for step in range(2):
        x_np = rng.standard_normal(shape).astype(np.float32)
        dy_np = rng.standard_normal(shape).astype(np.float32)
        x = torch.tensor(x_np, device="cuda", requires_grad=True)
        layer.zero_grad(set_to_none=True)
        out = layer(x, P.Mode.TRAIN)
        out.backward(torch.tensor(dy_np, device="cuda"))
        ref_out, cache, dx, dW, dg, db = O.train_step(p, x_np, dy_np)
        st = {kk: v.cpu().numpy() for kk, v in layer.last_state().items()}
        assert np.array_equal(st["w_q"], cache.w_q) if cfg.quantized else True
        assert_rel(layer.running_mean.cpu().numpy(), p.running_mean, 1e-10, "running_mean")
        assert_rel(layer.running_var.cpu().numpy(), p.running_var, 1e-10, "running_var")
        spikes_match_except_ties(out.detach().cpu().numpy(), ref_out, x_np, cache.w_q, cache.b_f, d)
        assert_close_scaled(x.grad.cpu().numpy(), dx, 1e-5, f"{name} step {step} dx")
        assert_close_scaled(layer.W.grad.cpu().numpy(), dW, 1e-5, f"{name} step {step} dW")
        assert_close_scaled(layer.gamma.grad.cpu().numpy(), dg, 1e-5, f"{name} step {step} dgamma")
        assert_close_scaled(layer.beta.grad.cpu().numpy(), db, 1e-5, f"{name} step {step} dbeta")


def test_bitwise_reproducible_run_to_run():
    """Fixed-order reductions, no floating-point atomics: two identical steps
    give bit-identical spikes, dx, gradients and running statistics (the
    reference is bit-reproducible, tests/test_train.py:70-82)."""
    P = _P()
    T, N, C, k, d = 1024, 64, 512, 4, 1
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn((T, N, C), generator=g, device="cuda")
    dy = torch.randn((T, N, C), generator=g, device="cuda")
    res = []
    for _ in range(2):
        cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
        layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(9), device="cuda")
        xi = x.clone().requires_grad_(True)
        out = layer(xi, P.Mode.TRAIN)
        out.backward(dy)
        torch.cuda.synchronize()
        res.append([t.detach().clone() for t in (out, xi.grad, layer.W.grad, layer.gamma.grad, layer.beta.grad,
                                                 layer.running_mean, layer.running_var)])
    for a, b in zip(*res):
        assert torch.equal(a, b)


def test_config1_full_parity():
    """T=250, B=32, C=128, k=4 (BASELINE config 1), every channel."""
    _oracle_subset_check(250, 32, 128, 4, 3, channels=list(range(128)), seed=11)


@pytest.mark.parametrize("k,d", [(8, 2), (16, 3), (16, 1)])
def test_high_order_parity(k, d):
    _oracle_subset_check(512, 16, 96, k, d, channels=[0, 31, 32, 63, 95], seed=k + d)


def test_bf16_io_parity():
    """bf16 I/O: oracle runs on the bf16 inputs widened to f32."""
    _oracle_subset_check(256, 16, 128, 2, 1, channels=[0, 5, 64, 127], dtype=torch.bfloat16, seed=5)


@pytest.mark.parametrize("k,d", [(4, 1), (4, 2)])
def test_bf16_io_parity_metric_shape(k, d):
    """bf16 I/O at the metric shape T=1024, B=64, C=512."""
    _oracle_subset_check(1024, 64, 512, k, d, channels=[0, 1, 200, 333, 511], dtype=torch.bfloat16, seed=7 + d)


def test_grads_accumulate_like_reference():
    """Two backward passes accumulate into .grad (reference uses +=)."""
    P = _P()
    cfg = P.NeuronConfig(channels=16, order=3, dilation=2, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(3), device="cuda")
    x = torch.randn(40, 4, 16, device="cuda")
    dy = torch.randn(40, 4, 16, device="cuda")
    layer(x, P.Mode.TRAIN).backward(dy)
    g1 = layer.W.grad.clone()
    layer(x, P.Mode.TRAIN).backward(dy)
    # second forward used updated running stats only for the running update;
    # batch-stat fusion makes both backward passes identical
    torch.testing.assert_close(layer.W.grad, 2 * g1, rtol=1e-12, atol=0)


def test_input_validation_errors():
    P = _P()
    layer = P.SpikingLayer(P.NeuronConfig(channels=4, order=2), device="cuda")
    with pytest.raises(ValueError):
        layer(torch.randn(5, 2, 3, device="cuda"), P.Mode.TRAIN)  # channel mismatch
    with pytest.raises(ValueError):
        layer(torch.randn(5, 4, device="cuda"), P.Mode.TRAIN)  # rank 2
    with pytest.raises(ValueError):
        layer(torch.randn(5, 2, 4), P.Mode.TRAIN)  # CPU tensor: no CPU fallback


@pytest.mark.parametrize("method", ["stream", "generic"])
@pytest.mark.parametrize("k,d", [(4, 2), (3, 1)])
def test_exact_threshold_ties_are_bit_exact(k, d, method):
    """Membranes exactly at / next to the threshold: integer inputs, running-stat
    fusion (b_f = beta exactly) and beta in {0, +-1e-45, -1e-46}.  The streamed
    forward decides spikes with an f32 filter and falls back to the exact f64
    membrane on ambiguous rows; every spike must equal the reference's, ties
    included (f32(h) >= 0, so h = -1e-46 spikes and h = -1e-45 does not)."""
    P = _P()
    T, N, C = 300, 20, 64
    rng = np.random.default_rng(7 + k)
    x_np = rng.integers(-2, 3, size=(T, N, C)).astype(np.float32)
    x_np[:, :, 48:] = 0.0  # whole streams at h2 = b_f
    dy_np = rng.standard_normal((T, N, C)).astype(np.float32)
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(k), device="cuda",
                           fuse_from_batch_stats=False)
    layer.configure(P.layer.LayerMethod(method))
    betas = np.array([0.0, -1e-45, -1e-46, 1e-45, 0.25, -0.25, 0.0, -1e-45] * (C // 8))
    with torch.no_grad():
        layer.beta.copy_(torch.tensor(betas, dtype=torch.float64))
    p = O.init_layer(C, k, d, weight_init="uniform", rng=np.random.default_rng(k), fuse_from_batch_stats=False)
    p.W = layer.W.detach().cpu().numpy().copy()
    p.beta = betas.copy()
    x = torch.tensor(x_np, device="cuda", requires_grad=True)
    out = layer(x, P.Mode.TRAIN)
    out.backward(torch.tensor(dy_np, device="cuda"))
    torch.cuda.synchronize()
    ref_out, cache, dx, dW, dg, db = O.train_step(p, x_np, dy_np)
    got = out.detach().cpu().numpy()
    assert np.array_equal(got, ref_out), f"{int((got != ref_out).sum())} spike mismatches at exact ties"
    assert_close_scaled(x.grad.cpu().numpy(), dx, 1e-5, "dx")
    assert_close_scaled(layer.W.grad.cpu().numpy(), dW, 1e-5, "dW")
    assert_close_scaled(layer.beta.grad.cpu().numpy(), db, 1e-5, "dbeta")


@pytest.mark.parametrize("teams,lag", [(2, 1), (3, 2), (5, 3), (10, 1)])
def test_cta_teams_and_lag_parity(monkeypatch, teams, lag):
    """Streamed schedule variants: nT CTA teams (uneven team sizes for 3 and 5 over
    148 SMs, one group per team for 10) and pipeline lags 1..3 give the same
    results as the reference."""
    monkeypatch.setenv("PSN_TEAMS", str(teams))
    monkeypatch.setenv("PSN_LAG", str(lag))
    _oracle_subset_check(400, 24, 320, 4, 2, channels=[0, 33, 97, 160, 255, 319], seed=teams * 10 + lag,
                         method="stream")


def _abi_step(P, L, x, dy, layer, desc, ws):
    """One fwd+bwd through the C ABI on a caller-provided workspace."""
    import ctypes
    C, k = x.shape[2], desc.k
    out, dx = torch.empty_like(x), torch.empty_like(x)
    fold = torch.empty((C, L.fold_stride(k)), dtype=torch.float64, device=x.device)
    dW = torch.empty((C, k), dtype=torch.float64, device=x.device)
    dg, db = torch.empty(C, dtype=torch.float64, device=x.device), torch.empty(C, dtype=torch.float64, device=x.device)
    rm, rv = layer.running_mean.clone(), layer.running_var.clone()
    sp = torch.cuda.current_stream().cuda_stream
    lib = L.lib()
    L.check(lib.psn_forward_train(ctypes.byref(desc), x.data_ptr(), layer.W.data_ptr(), layer.gamma.data_ptr(),
                                  layer.beta.data_ptr(), rm.data_ptr(), rv.data_ptr(), out.data_ptr(),
                                  fold.data_ptr(), ws.data_ptr(), sp))
    L.check(lib.psn_backward(ctypes.byref(desc), x.data_ptr(), dy.data_ptr(), layer.W.data_ptr(),
                             layer.gamma.data_ptr(), fold.data_ptr(), dx.data_ptr(), dW.data_ptr(), dg.data_ptr(),
                             db.data_ptr(), ws.data_ptr(), sp))
    torch.cuda.synchronize()
    return [t.cpu() for t in (out, dx, dW, dg, db, rm, rv)]


@pytest.mark.parametrize("route", ["stream", "auto"])
def test_workspace_reuse_garbage_and_alternating_geometries(route):
    """Workspace contract: any content is fine.  Repeated calls, a garbage-filled
    buffer and a buffer alternating between two geometries must all give the
    same results as a fresh zeroed workspace (streamed kernels, and the
    planner's choice at these sizes: the generic ones)."""
    P = _P()
    from paper_2501_14490_b200 import _lib as L
    shapes = [(300, 20, 128), (257, 12, 64)]
    runs = []
    for T, N, C in shapes:
        cfg = P.NeuronConfig(channels=C, order=4, dilation=2, quantized=True)
        layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(C), device="cuda")
        x = torch.randn((T, N, C), device="cuda")
        dy = torch.randn((T, N, C), device="cuda")
        extra = L.PSN_STREAM if route == "stream" else 0
        desc = L.make_desc(x.shape, 4, 2, torch.float32, flags=L.PSN_QUANTIZED | L.PSN_USE_BATCH_STATS | extra)
        assert L.plan_info(desc, True)["streamed"] == (1 if route == "stream" else 0)
        runs.append((x, dy, layer, desc))
    nbytes = max(int(L.lib().psn_workspace_bytes(__import__("ctypes").byref(r[3]))) for r in runs)
    refs = [_abi_step(P, L, x, dy, layer, desc, torch.zeros(nbytes, dtype=torch.uint8, device="cuda"))
            for x, dy, layer, desc in runs]

    def same(got, ref):  # bitwise: fixed-order reductions, no atomics
        for g, r in zip(got, ref):
            assert torch.equal(g, r)

    shared = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda")  # garbage
    for rep in range(3):
        for (x, dy, layer, desc), ref in zip(runs, refs):
            same(_abi_step(P, L, x, dy, layer, desc, shared), ref)


@pytest.mark.parametrize("route", ["stream", "auto"])
def test_cuda_graph_capture_replays_the_step(route):
    """The C-ABI calls are stream-ordered and allocation-free, so one fwd+bwd
    step captures into a CUDA graph; replays give the direct results."""
    import ctypes
    P = _P()
    from paper_2501_14490_b200 import _lib as L
    T, N, C, k, d = 300, 20, 128, 4, 2
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(3), device="cuda")
    x = torch.randn((T, N, C), device="cuda")
    dy = torch.randn((T, N, C), device="cuda")
    extra = L.PSN_STREAM if route == "stream" else 0
    desc = L.make_desc(x.shape, k, d, torch.float32, flags=L.PSN_QUANTIZED | L.PSN_USE_BATCH_STATS | extra)
    ws = L.workspace(desc, x.device)
    out, dx = torch.empty_like(x), torch.empty_like(x)
    fold = torch.empty((C, L.fold_stride(k)), dtype=torch.float64, device="cuda")
    dW = torch.empty((C, k), dtype=torch.float64, device="cuda")
    dg, db = torch.empty(C, dtype=torch.float64, device="cuda"), torch.empty(C, dtype=torch.float64, device="cuda")
    rm0, rv0 = layer.running_mean.clone(), layer.running_var.clone()
    lib = L.lib()

    def step(stream):
        L.check(lib.psn_forward_train(ctypes.byref(desc), x.data_ptr(), layer.W.data_ptr(), layer.gamma.data_ptr(),
                                      layer.beta.data_ptr(), layer.running_mean.data_ptr(),
                                      layer.running_var.data_ptr(), out.data_ptr(), fold.data_ptr(),
                                      ws.data_ptr(), stream))
        L.check(lib.psn_backward(ctypes.byref(desc), x.data_ptr(), dy.data_ptr(), layer.W.data_ptr(),
                                 layer.gamma.data_ptr(), fold.data_ptr(), dx.data_ptr(), dW.data_ptr(),
                                 dg.data_ptr(), db.data_ptr(), ws.data_ptr(), stream))

    step(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = [t.clone() for t in (out, dx, dW, dg, db)]
    ref_stats = (layer.running_mean.clone(), layer.running_var.clone())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(torch.cuda.current_stream().cuda_stream)
    for t in (out, dx, dW, dg, db):
        t.zero_()
    layer.running_mean.copy_(rm0)
    layer.running_var.copy_(rv0)
    g.replay()
    torch.cuda.synchronize()
    for got, want in zip((out, dx, dW, dg, db), ref):
        assert torch.equal(got, want)
    assert torch.equal(layer.running_mean, ref_stats[0])
    assert torch.equal(layer.running_var, ref_stats[1])


@pytest.mark.parametrize("method", ["stream", "generic"])
@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("k", list(range(1, 17)))
def test_order_dilation_sweep(k, d, method):
    """Every order 1..16 at every sawtooth dilation, on both kernel families
    (the streamed method falls back to the generic kernels where the shape
    does not qualify: k > 8), every channel against the oracle; T off the
    time-tile grid, B off the batch-tile grid."""
    _oracle_subset_check(203, 11, 64, k, d, channels=list(range(64)), seed=1000 + 10 * k + d, method=method)


@pytest.mark.parametrize("method", ["stream", "generic"])
@pytest.mark.parametrize("k,d", [(2, 1), (4, 3), (8, 2), (16, 1), (16, 3)])
def test_bf16_order_sweep(k, d, method):
    """bf16 I/O across orders and dilations on both kernel families (bf16 dx
    bound: half a bf16 ulp plus the f32 bound)."""
    _oracle_subset_check(150, 9, 96, k, d, channels=list(range(96)), dtype=torch.bfloat16, seed=2000 + 10 * k + d,
                         method=method)


@pytest.mark.parametrize("method", ["stream", "generic"])
@pytest.mark.parametrize("shape,k,d", [((5, 1, 1), 16, 3), ((1, 3, 5), 1, 1), ((2, 2, 33), 4, 2),
                                        ((40, 1, 3, 7), 5, 2), ((17, 2, 2, 5, 3), 3, 3), ((64, 33, 37), 2, 1)])
def test_odd_shapes(shape, k, d, method):
    """Degenerate and ragged extents on both kernel families: T = 1, T < halo,
    N = 1, C = 1, J not a multiple of the 16-byte piece, odd spatial axes."""
    T, N, C = shape[:3]
    _oracle_subset_check(T, N, C, k, d, channels=list(range(C)), seed=sum(shape) + 3 * k + d, spatial=shape[3:],
                         method=method)


@pytest.mark.parametrize("method", ["auto", "generic"])
def test_float64_carrier_medium_shape(method):
    """float64 carrier (generic kernels: 8-byte ring elements, 16-byte pieces of
    two columns) at a medium shape, every channel against the oracle run on
    the same f64 inputs; f64 tolerance."""
    P = _P()
    T, N, C, k, d = 200, 9, 64, 4, 2
    rng = np.random.default_rng(77)
    x_np = rng.standard_normal((T, N, C))
    dy_np = rng.standard_normal((T, N, C))
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(78), device="cuda")
    layer.configure(P.layer.LayerMethod(method))
    x = torch.tensor(x_np, device="cuda", requires_grad=True)
    out = layer(x, P.Mode.TRAIN)
    out.backward(torch.tensor(dy_np, device="cuda"))
    p = O.init_layer(C, k, d, weight_init="uniform", rng=np.random.default_rng(78))
    p.W = layer.W.detach().cpu().numpy()
    ref_out, cache, dx, dW, dg, db = O.train_step(p, x_np, dy_np)
    spikes_match_except_ties(out.detach().cpu().numpy(), ref_out, x_np, cache.w_q, cache.b_f, d)
    assert_close_scaled(x.grad.cpu().numpy(), dx, 1e-9, "dx")
    assert_close_scaled(layer.W.grad.cpu().numpy(), dW, 1e-9, "dW")
    assert_close_scaled(layer.gamma.grad.cpu().numpy(), dg, 1e-9, "dgamma")
    assert_close_scaled(layer.beta.grad.cpu().numpy(), db, 1e-9, "dbeta")


@pytest.mark.parametrize("method", ["auto", "generic"])
def test_smooth_mode_medium_shape(method):
    """SMOOTH mode (spike primitive output, statistics frozen; generic kernels)
    at a medium shape against the oracle."""
    P = _P()
    T, N, C, k, d = 150, 8, 96, 3, 3
    rng = np.random.default_rng(88)
    x_np = rng.standard_normal((T, N, C)).astype(np.float32)
    dy_np = rng.standard_normal((T, N, C)).astype(np.float32)
    cfg = P.NeuronConfig(channels=C, order=k, dilation=d, quantized=True)
    layer = P.SpikingLayer(cfg, weight_init="uniform", rng=np.random.default_rng(89), device="cuda")
    layer.configure(P.layer.LayerMethod(method))
    x = torch.tensor(x_np, device="cuda", requires_grad=True)
    out = layer(x, P.Mode.SMOOTH)
    out.backward(torch.tensor(dy_np, device="cuda"))
    p = O.init_layer(C, k, d, weight_init="uniform", rng=np.random.default_rng(89))
    p.W = layer.W.detach().cpu().numpy()
    ref_out, cache = O.forward_train(p, x_np, smooth=True)
    dx, dW, dg, db = O.backward(p, cache, dy_np)
    assert_close_scaled(out.detach().cpu().numpy(), ref_out, 1e-6, "smooth output")
    assert_close_scaled(x.grad.cpu().numpy(), dx, 1e-5, "dx")
    assert_close_scaled(layer.W.grad.cpu().numpy(), dW, 1e-5, "dW")
    assert_close_scaled(layer.gamma.grad.cpu().numpy(), dg, 1e-5, "dgamma")
    assert_close_scaled(layer.beta.grad.cpu().numpy(), db, 1e-5, "dbeta")

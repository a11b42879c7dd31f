"""Generate the golden fixtures that pin ``oracle/psn_oracle.py`` (and through
it the CUDA path) to the reference implementation.

Run IN THE BUILD CONTAINER ONLY (it imports the read-only reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Every array written here is produced by the reference's own code
(shiftsnn.network.SpikingLayer, shiftsnn.engines, shiftsnn.quant): inputs are
seeded numpy draws, outputs are what the reference returns.  The fixtures are
small (a few hundred KB total) and committed next to this script.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import shiftsnn  # noqa: F401
    from shiftsnn import engines, network, neuron, quant, surrogate, tensor
    return engines, network, neuron, quant, surrogate, tensor


# One entry per layer fixture.  Shapes are time-first [T, N, C, *spatial].
LAYER_CASES = [
    # name, shape, k, d, extra flags
    ("k4d1", (40, 6, 16), 4, 1, {}),
    ("k4d2", (40, 6, 16), 4, 2, {}),
    ("k4d3", (40, 6, 16), 4, 3, {}),
    ("k2d1_lif", (25, 4, 8), 2, 1, {"weight_init": "lif"}),
    ("k1d1", (12, 3, 5), 1, 1, {}),
    ("k16d3", (64, 3, 12), 16, 3, {}),
    ("k8d2_T_lt_halo", (9, 2, 7), 8, 2, {}),
    ("k5d1_float", (30, 4, 9), 5, 1, {"quantized": False}),
    ("k3d2_shared", (30, 4, 9), 3, 2, {"shared": True}),
    ("k4d1_running", (30, 4, 9), 4, 1, {"fuse_from_batch_stats": False}),
    ("k4d1_roundste", (30, 4, 9), 4, 1, {"grad_mode": "round_ste"}),
    ("k4d2_rational", (30, 4, 9), 4, 2, {"surrogate": ("rational", 10.0)}),
    ("k4d1_smooth", (30, 4, 9), 4, 1, {"smooth": True}),
    ("k4d1_smooth_q", (30, 4, 9), 4, 1, {"smooth": True, "quantize_in_smooth_mode": True}),
    ("k2d1_spatial4", (10, 3, 4, 6), 2, 1, {}),
    ("k3d2_spatial5", (8, 2, 3, 3, 4), 3, 2, {}),
    ("k4d1_f64", (30, 4, 9), 4, 1, {"dtype": "float64"}),
    ("k4d3_cfg1_small", (64, 8, 32), 4, 3, {}),
]


def make_layer_case(ref, name, shape, k, d, flags, seed):
    engines, network, neuron, quant, surrogate, tensor = ref
    dtype = np.dtype(flags.get("dtype", "float32"))
    rng = np.random.default_rng(seed)
    C = shape[2]
    sharing = neuron.WeightSharing.SHARED if flags.get("shared") else neuron.WeightSharing.CHANNEL_WISE
    grad_mode = (quant.QuantGradMode.ROUND_STE if flags.get("grad_mode") == "round_ste"
                 else quant.QuantGradMode.WHOLE_STE)
    cfg = neuron.NeuronConfig(channels=C, order=k, dilation=d, weight_sharing=sharing,
                              quantized=flags.get("quantized", True), grad_mode=grad_mode)
    kind, alpha = flags.get("surrogate", ("arctan", 2.0))
    sur = surrogate.SurrogateConfig(surrogate.SurrogateKind(kind), alpha)
    layer = network.SpikingLayer(cfg, surrogate=sur,
                                 weight_init=flags.get("weight_init", "uniform"),
                                 rng=np.random.default_rng(seed + 1),
                                 fuse_from_batch_stats=flags.get("fuse_from_batch_stats", True))
    layer.quantize_in_smooth_mode = bool(flags.get("quantize_in_smooth_mode", False))
    # non-trivial gamma/beta/running stats so every term of the fold matters
    layer.gamma.value[...] = rng.uniform(0.5, 1.5, C)
    layer.beta.value[...] = rng.uniform(-1.5, -0.5, C)
    layer.thr.running_mean[...] = rng.normal(0.0, 0.1, C)
    layer.thr.running_var[...] = rng.uniform(0.5, 1.5, C)
    mode = network.Mode.SMOOTH if flags.get("smooth") else network.Mode.TRAIN

    out = {
        "W": layer.W.value.copy(), "gamma": layer.gamma.value.copy(),
        "beta": layer.beta.value.copy(),
        "running_mean_in": layer.thr.running_mean.copy(),
        "running_var_in": layer.thr.running_var.copy(),
    }
    for step in range(2):
        x = rng.standard_normal(shape).astype(dtype)
        dy = rng.standard_normal(shape).astype(dtype)
        for p in layer.parameters():
            p.grad[...] = 0.0
        y = layer.forward(tensor.TemporalTensor(x, tensor.Layout.TIME_FIRST), mode)
        c = layer._cache
        dx = layer.backward(tensor.TemporalTensor(dy, tensor.Layout.TIME_FIRST))
        pre = f"s{step}_"
        out.update({
            pre + "x": x, pre + "dy": dy, pre + "out": y.data,
            pre + "h1": c["h1"].data, pre + "h2": c["h2"].data,
            pre + "mu": np.asarray(c["mu"]), pre + "s": np.asarray(c["s"]),
            pre + "a": np.asarray(c["a"]), pre + "w_f": np.asarray(c["w_f"]),
            pre + "w_q": np.asarray(c["w_q"]),
            pre + "running_mean": layer.thr.running_mean.copy(),
            pre + "running_var": layer.thr.running_var.copy(),
            pre + "dx": dx.data, pre + "dW": layer.W.grad.copy(),
            pre + "dgamma": layer.gamma.grad.copy(), pre + "dbeta": layer.beta.grad.copy(),
        })
        # b_f is not cached by the reference; it is beta - a*mu (network.py:255)
        out[pre + "b_f"] = layer.beta.value - np.asarray(c["a"]) * np.asarray(c["mu"])
    # EVAL forward with the running stats after the two steps (network.py:219-234)
    xe = rng.standard_normal(shape).astype(dtype)
    ye = layer.forward(tensor.TemporalTensor(xe, tensor.Layout.TIME_FIRST), network.Mode.EVAL)
    out["eval_x"] = xe
    out["eval_out"] = ye.data
    meta = {"name": name, "shape": list(shape), "k": k, "d": d, "flags": {
        kk: (list(v) if isinstance(v, tuple) else v) for kk, v in flags.items()},
        "mode": mode.value, "dtype": str(dtype), "seed": seed}
    return out, meta


def make_quant_case(ref):
    engines, network, neuron, quant, surrogate, tensor = ref
    rng = np.random.default_rng(100)
    vals = [np.exp2(rng.uniform(-18.0, 17.0, 20000)) * rng.choice([-1.0, 1.0], 20000)]
    mids = []
    for e in range(-20, 19):
        mid = math.sqrt(2.0) * 2.0 ** e
        for v in (np.nextafter(mid, 0.0), mid, np.nextafter(mid, np.inf)):
            mids += [v, -v]
        p2 = 2.0 ** e
        mids += [p2, np.nextafter(p2, 0.0), np.nextafter(p2, np.inf)]
    vals.append(np.array(mids))
    vals.append(np.array([0.0, -0.0, 0.5, -0.3, 0.75, 2.0 ** 25, 2.0 ** -25,
                          5e-324, 1e-310, 1.7e308, -1.7e308]))
    w = np.concatenate(vals)
    q = quant.quantize_pow2(w)
    g = rng.standard_normal(w.shape)
    ste = quant.quantize_backward(g, w, quant.QuantGradMode.ROUND_STE)
    quant.reset_instability_count()
    return {"w": w, "sign": q.sign, "exponent": q.exponent, "g": g, "round_ste": ste}


def make_engine_case(ref):
    """Random small instances of every engine entry point on the path."""
    engines, network, neuron, quant, surrogate, tensor = ref
    TT = tensor.TemporalTensor
    TF = tensor.Layout.TIME_FIRST
    rng = np.random.default_rng(200)
    out = {}
    n = 0
    for _ in range(40):
        T = int(rng.integers(1, 17)); k = int(rng.integers(1, 9)); d = int(rng.integers(1, 4))
        C = int(rng.integers(1, 9)); N = int(rng.integers(1, 5))
        dt = np.float32 if rng.integers(2) else np.float64
        x = rng.standard_normal((T, N, C)).astype(dt)
        rows = 1 if rng.integers(4) == 0 else C
        w = rng.standard_normal((rows, k))
        b = rng.standard_normal(C) if rng.integers(2) else None
        dh = rng.standard_normal((T, N, C)).astype(dt)
        sign = rng.choice([-1, 0, 1], size=(C, k)).astype(np.int8)
        expo = rng.integers(-16, 16, size=(C, k)).astype(np.int8)
        sw = quant.ShiftWeights(sign=sign, exponent=expo)
        p = f"e{n}_"
        out[p + "x"] = x; out[p + "w"] = w; out[p + "dh"] = dh
        out[p + "d"] = np.array(d)
        if b is not None:
            out[p + "b"] = b
        out[p + "fwd"] = engines.conv_forward_direct(TT(x, TF), w, bias=b, d=d).data
        out[p + "sign"] = sign; out[p + "exponent"] = expo
        out[p + "shift"] = engines.conv_forward_shift(TT(x, TF), sw, bias=b, d=d).data
        out[p + "bwd_in"] = engines.conv_backward_input(TT(dh, TF), w, d).data
        xw = x if rows == C else x  # weight grad takes x of any rows
        out[p + "bwd_w"] = engines.conv_backward_weight(TT(xw, TF), TT(dh, TF), k, d,
                                                       shared=(rows == 1))
        out[p + "bwd_b"] = engines.conv_backward_bias(TT(dh, TF))
        # int32 fixed-point carrier
        xi = rng.integers(-(2 ** 20), 2 ** 20, size=(T, N, C)).astype(np.int32)
        quant.reset_saturation_count()
        out[p + "xi"] = xi
        bi = rng.integers(-1000, 1000, C).astype(np.float64) + 0.5 if b is not None else None
        if bi is not None:
            out[p + "bi"] = bi
        out[p + "shift_int"] = engines.conv_forward_shift(TT(xi, TF), sw, bias=bi, d=d).data
        out[p + "shift_int_sat"] = np.array(quant.saturation_count())
        n += 1
    out["count"] = np.array(n)
    quant.reset_saturation_count()
    return out


def main():
    ref = _import_reference()
    manifest = []
    for i, (name, shape, k, d, flags) in enumerate(LAYER_CASES):
        arrays, meta = make_layer_case(ref, name, shape, k, d, flags, seed=1000 + 17 * i)
        np.savez_compressed(os.path.join(HERE, f"layer_{name}.npz"), **arrays)
        manifest.append(meta)
    np.savez_compressed(os.path.join(HERE, "quant.npz"), **make_quant_case(ref))
    np.savez_compressed(os.path.join(HERE, "engines.npz"), **make_engine_case(ref))
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump({"source": "reference shiftsnn 0.1.0 at /root/reference/pkg/src",
                   "numpy": np.__version__, "layer_cases": manifest}, f, indent=1)
    print(f"wrote {len(manifest)} layer fixtures + quant + engines to {HERE}")


if __name__ == "__main__":
    main()

"""Pin the CPU oracle to the reference: every oracle function is compared
bit-for-bit against fixtures produced by running the reference itself
(tests/golden/make_golden.py), and against the reference's own known-answer
tests.  CPU only."""

import glob
import json
import math
import os

import numpy as np
import pytest

from oracle import psn_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))
CASES = {c["name"]: c for c in MANIFEST["layer_cases"]}


def _params(z, meta):
    f = meta["flags"]
    kind, alpha = f.get("surrogate", ["arctan", 2.0])
    return O.LayerParams(
        W=z["W"].copy(), gamma=z["gamma"].copy(), beta=z["beta"].copy(),
        running_mean=z["running_mean_in"].copy(), running_var=z["running_var_in"].copy(),
        d=meta["d"], quantized=f.get("quantized", True),
        round_ste=f.get("grad_mode") == "round_ste",
        fuse_from_batch_stats=f.get("fuse_from_batch_stats", True),
        quantize_in_smooth_mode=f.get("quantize_in_smooth_mode", False),
        surrogate=kind, alpha=alpha)


def _eq(a, b, what):
    a = np.asarray(a); b = np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    assert a.dtype == b.dtype, (what, a.dtype, b.dtype)
    assert np.array_equal(a, b), f"{what}: max |diff| {np.max(np.abs(a.astype(float) - b.astype(float)))}"


@pytest.mark.parametrize("name", sorted(CASES))
def test_layer_fixture_bit_exact(name):
    meta = CASES[name]
    z = np.load(os.path.join(GOLDEN, f"layer_{name}.npz"))
    p = _params(z, meta)
    smooth = meta["mode"] == "smooth"
    for step in range(2):
        pre = f"s{step}_"
        out, c = O.forward_train(p, z[pre + "x"], smooth=smooth)
        _eq(c.h1, z[pre + "h1"], "h1")
        _eq(c.h2, z[pre + "h2"], "h2")
        _eq(c.mu, z[pre + "mu"], "mu")
        _eq(c.s, z[pre + "s"], "s")
        _eq(c.w_f, z[pre + "w_f"], "w_f")
        _eq(c.w_q, z[pre + "w_q"], "w_q")
        _eq(c.b_f, z[pre + "b_f"], "b_f")
        _eq(out, z[pre + "out"], "spikes")
        _eq(p.running_mean, z[pre + "running_mean"], "running_mean")
        _eq(p.running_var, z[pre + "running_var"], "running_var")
        dx, dW, dg, db = O.backward(p, c, z[pre + "dy"])
        _eq(dx, z[pre + "dx"], "dx")
        _eq(dW, z[pre + "dW"], "dW")
        _eq(dg, z[pre + "dgamma"], "dgamma")
        _eq(db, z[pre + "dbeta"], "dbeta")
    _eq(O.forward_eval(p, z["eval_x"]), z["eval_out"], "eval spikes")


def test_quantizer_matches_reference_sweep():
    z = np.load(os.path.join(GOLDEN, "quant.npz"))
    sign, expo = O.quantize_pow2(z["w"])
    _eq(sign, z["sign"], "sign")
    _eq(expo, z["exponent"], "exponent")
    with np.errstate(over="ignore"):
        _eq(O.quantize_backward(z["g"], z["w"], round_ste=True), z["round_ste"], "round_ste")


def test_engines_match_reference_instances():
    z = np.load(os.path.join(GOLDEN, "engines.npz"))
    for n in range(int(z["count"])):
        p = f"e{n}_"
        x, w, dh, d = z[p + "x"], z[p + "w"], z[p + "dh"], int(z[p + "d"])
        b = z[p + "b"] if p + "b" in z else None
        _eq(O.conv_forward(x, w, b, d), z[p + "fwd"], "conv_forward")
        shift_w = O.dequantize(z[p + "sign"], z[p + "exponent"])
        _eq(O.conv_forward(x, shift_w, b, d), z[p + "shift"], "shift float")
        _eq(O.conv_backward_input(dh, w, d), z[p + "bwd_in"], "bwd input")
        _eq(O.conv_backward_weight(x, dh, w.shape[1], d, shared=w.shape[0] == 1),
            z[p + "bwd_w"], "bwd weight")
        _eq(O.conv_backward_bias(dh), z[p + "bwd_b"], "bwd bias")
        bi = z[p + "bi"] if p + "bi" in z else None
        got, sat = O.conv_forward_shift_int(z[p + "xi"], z[p + "sign"], z[p + "exponent"], bi, d)
        _eq(got, z[p + "shift_int"], "shift int")
        assert sat == int(z[p + "shift_int_sat"])


# ---- the reference's own known-answer tests ---------------

def _tt(seq):
    return np.asarray(seq, dtype=np.float64)[:, None, None]


def test_kat_charge():
    # reference tests/test_engines.py:101-108, tests/test_neuron.py:53-65
    assert O.conv_forward(_tt([1, 0, 1]), np.array([[0.5, 1.0]]), d=1).ravel().tolist() == [1.0, 0.5, 1.0]
    assert O.conv_forward(_tt([1, 2, 3, 4]), np.array([[1.0, 1.0]]), d=2).ravel().tolist() == [1, 2, 4, 6]
    x = _tt([3.0, -1.0, 2.0])
    assert np.array_equal(O.conv_forward(x, np.array([[1.0]])), x)


def test_kat_shift_int():
    # reference tests/test_engines.py:148-167
    x = np.array([8, 16, -32, 64], dtype=np.int32)[:, None, None]
    h, sat = O.conv_forward_shift_int(x, np.array([[1, -1]]), np.array([[-2, 1]]), d=1)
    assert h.dtype == np.int32 and h.ravel().tolist() == [-16, -30, 68, -136] and sat == 0
    h, sat = O.conv_forward_shift_int(np.full((1, 1, 1), 2 ** 28, dtype=np.int32),
                                      np.array([[1]]), np.array([[5]]))
    assert h.ravel()[0] == np.iinfo(np.int32).max and sat == 1


def test_kat_backward():
    # reference tests/test_engines.py:175-216
    assert O.conv_backward_input(_tt([1.0, -2.0, 3.0]), np.array([[0.5]])).ravel().tolist() == [0.5, -1.0, 1.5]
    w0, w1 = 2.0, 5.0
    assert O.conv_backward_input(_tt([1.0, 10.0]), np.array([[w0, w1]])).ravel().tolist() == [w1 + w0 * 10, w1 * 10]
    assert np.array_equal(O.conv_backward_weight(_tt([0.0] * 3), _tt([1.0] * 3), k=2), np.zeros((1, 2)))
    assert np.array_equal(O.conv_backward_weight(_tt([3.0]), _tt([2.0]), k=1), [[6.0]])
    assert np.array_equal(O.conv_backward_bias(np.ones((3, 2, 1))), [6.0])


def test_kat_quantizer():
    # reference tests/test_quant.py:30-85
    def q1(w):
        s, e = O.quantize_pow2(np.array([[w]]))
        return int(s[0, 0]), int(e[0, 0]), float(O.dequantize(s, e)[0, 0])
    assert q1(0.5) == (1, -1, 0.5)
    assert q1(-0.3) == (-1, -2, -0.25)
    assert q1(0.75) == (1, 0, 1.0)
    assert q1(0.0) == (0, 0, 0.0)
    for e in (-12, -3, 0, 5, 11):
        mid = math.sqrt(2.0) * 2.0 ** e
        assert q1(np.nextafter(mid, 0.0))[1] == e
        assert q1(np.nextafter(mid, np.inf))[1] == e + 1
    assert q1(2.0 ** 25)[1] == O.E_MAX
    assert q1(2.0 ** -25)[1] == O.E_MIN
    with pytest.raises(ValueError):
        O.quantize_pow2(np.array([np.inf]))
    g = np.ones((1, 2))
    np.testing.assert_allclose(O.quantize_backward(g, np.array([[0.75, 0.5]]), True), [[4 / 3, 1.0]], rtol=1e-15)


def test_kat_surrogate_and_schedule():
    # reference tests/test_network.py:20-28, tests/test_neuron.py:37-50, 233-237
    assert O.spike_backward(0.0, O.ARCTAN, 2.0) == pytest.approx(1.0)
    assert O.spike_backward(0.0, O.RATIONAL, 10.0) == pytest.approx(1.0)
    assert O.sawtooth_schedule(6) == [1, 2, 3, 1, 2, 3]
    assert O.receptive_field([2, 2, 2], [1, 2, 3]) == 7
    np.testing.assert_allclose(O.lif_taps(3, 2.0), [0.125, 0.25, 0.5], rtol=1e-15)


def test_kat_bn_fold_substitution():
    # reference tests/test_neuron.py:140-145: gamma=2, var=3, eps=1, mean=1 -> W_f=[1,1], b_f=-1
    p = O.LayerParams(W=np.array([[1.0, 1.0]]), gamma=np.array([2.0]), beta=np.array([0.0]),
                      running_mean=np.array([1.0]), running_var=np.array([3.0]), eps=1.0)
    w_f, b_f = O.fused_running(p)
    assert np.array_equal(w_f, [[1.0, 1.0]]) and np.array_equal(b_f, [-1.0])


def test_quantizer_property_sweep():
    # reference tests/test_acceptance.py:218-234 (criterion 7), 2e5 draws here
    rng = np.random.default_rng(3)
    w = np.exp2(rng.uniform(-16.4, 15.4, 200_000)) * rng.choice([-1.0, 1.0], 200_000)
    s, e = O.quantize_pow2(w)
    v = O.dequantize(s, e)
    s2, e2 = O.quantize_pow2(v)
    assert np.array_equal(s, s2) and np.array_equal(e, e2)
    sn, en = O.quantize_pow2(-w)
    assert np.array_equal(sn, -s) and np.array_equal(en, e)
    r = v / w
    assert np.all((r >= 2 ** -0.5) & (r <= 2 ** 0.5))

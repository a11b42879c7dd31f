"""GPU engine-level operators vs the reference's own outputs (golden fixtures)
and known-answer tests (reference tests/test_engines.py, tests/test_quant.py)."""

import math
import os

import numpy as np
import pytest
import torch

from tests.parity import assert_close_scaled

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _P():
    import paper_2501_14490_b200 as P
    return P


def _t(a):
    return torch.tensor(np.asarray(a), device="cuda")


def test_engine_instances_bit_exact():
    P = _P()
    z = np.load(os.path.join(GOLDEN, "engines.npz"))
    for n in range(int(z["count"])):
        p = f"e{n}_"
        x, w, dh, d = z[p + "x"], z[p + "w"], z[p + "dh"], int(z[p + "d"])
        b = z[p + "b"] if p + "b" in z else None
        k = w.shape[1]
        got = P.conv_forward(_t(x), _t(w), None if b is None else _t(b), d).cpu().numpy()
        assert got.dtype == z[p + "fwd"].dtype and np.array_equal(got, z[p + "fwd"]), f"fwd {n}"
        sw = P.ShiftWeights(_t(z[p + "sign"]), _t(z[p + "exponent"]))
        got = P.conv_forward(_t(x), sw, None if b is None else _t(b), d).cpu().numpy()
        assert np.array_equal(got, z[p + "shift"]), f"shift {n}"
        got = P.conv_backward_input(_t(dh), _t(w), d).cpu().numpy()
        assert np.array_equal(got, z[p + "bwd_in"]), f"bwd_in {n}"
        got = P.conv_backward_weight(_t(x), _t(dh), k, d, shared=w.shape[0] == 1).cpu().numpy()
        assert_close_scaled(got, z[p + "bwd_w"], 1e-12, f"bwd_w {n}")
        got = P.conv_backward_bias(_t(dh)).cpu().numpy()
        assert_close_scaled(got, z[p + "bwd_b"], 1e-12, f"bwd_b {n}")
        bi = z[p + "bi"] if p + "bi" in z else None
        got, sat = P.conv_forward_shift_int(_t(z[p + "xi"]), sw, None if bi is None else _t(bi), d)
        assert np.array_equal(got.cpu().numpy(), z[p + "shift_int"]), f"shift_int {n}"
        assert sat == int(z[p + "shift_int_sat"])


def test_quantizer_matches_reference_sweep():
    P = _P()
    z = np.load(os.path.join(GOLDEN, "quant.npz"))
    q = P.quantize_pow2(_t(z["w"]))
    assert np.array_equal(q.sign.cpu().numpy(), z["sign"])
    assert np.array_equal(q.exponent.cpu().numpy(), z["exponent"])


def _tt(seq, dtype=torch.float64):
    return torch.tensor(seq, dtype=dtype, device="cuda")[:, None, None]


def test_kat_charge_and_backward():
    P = _P()
    # reference tests/test_engines.py:101-108, 175-216
    assert P.conv_forward(_tt([1, 0, 1]), _t([[0.5, 1.0]]), d=1).flatten().tolist() == [1.0, 0.5, 1.0]
    assert P.conv_forward(_tt([1, 2, 3, 4]), _t([[1.0, 1.0]]), d=2).flatten().tolist() == [1, 2, 4, 6]
    assert P.conv_backward_input(_tt([1.0, -2.0, 3.0]), _t([[0.5]])).flatten().tolist() == [0.5, -1.0, 1.5]
    assert P.conv_backward_input(_tt([1.0, 10.0]), _t([[2.0, 5.0]])).flatten().tolist() == [25.0, 50.0]
    assert P.conv_backward_weight(_tt([3.0]), _tt([2.0]), k=1).tolist() == [[6.0]]
    assert P.conv_backward_bias(torch.ones(3, 2, 1, dtype=torch.float64, device="cuda")).tolist() == [6.0]


def test_kat_shift_int_and_saturation():
    P = _P()
    x = torch.tensor([8, 16, -32, 64], dtype=torch.int32, device="cuda")[:, None, None]
    sw = P.ShiftWeights(_t([[1, -1]]), _t([[-2, 1]]))
    h, sat = P.conv_forward_shift_int(x, sw, d=1)
    assert h.dtype == torch.int32 and h.flatten().tolist() == [-16, -30, 68, -136] and sat == 0
    x = torch.full((1, 1, 1), 2 ** 28, dtype=torch.int32, device="cuda")
    h, sat = P.conv_forward_shift_int(x, P.ShiftWeights(_t([[1]]), _t([[5]])), d=1)
    assert h.item() == 2 ** 31 - 1 and sat == 1


def test_kat_quantizer():
    P = _P()
    def q1(w):
        q = P.quantize_pow2(_t([[w]]))
        return int(q.sign.item()), int(q.exponent.item()), float(P.dequantize(q).item())
    assert q1(0.5) == (1, -1, 0.5)
    assert q1(-0.3) == (-1, -2, -0.25)
    assert q1(0.75) == (1, 0, 1.0)
    assert q1(0.0) == (0, 0, 0.0)
    for e in (-12, -3, 0, 5, 11):
        mid = math.sqrt(2.0) * 2.0 ** e
        assert q1(float(np.nextafter(mid, 0.0)))[1] == e
        assert q1(float(np.nextafter(mid, np.inf)))[1] == e + 1
    assert q1(2.0 ** 25)[1] == 15 and q1(2.0 ** -25)[1] == -16
    with pytest.raises(ValueError):
        P.quantize_pow2(_t([float("inf")]))


def test_engine_errors_mirror_reference():
    P = _P()
    x = _tt([1.0, 2.0])
    with pytest.raises(ValueError):
        P.conv_forward(x, _t(np.ones((3, 2))))  # channel mismatch
    with pytest.raises(ValueError):
        P.conv_forward(x, _t(np.ones((1, 2))), bias=_t(np.ones(2)))
    with pytest.raises(ValueError):
        P.conv_forward(x, _t(np.ones((1, 2))), d=0)
    with pytest.raises(TypeError):
        P.conv_forward_shift(x, _t(np.ones((1, 1))))


@pytest.mark.parametrize("shape", [(6, 2, 3, 4), (5, 2, 3, 2, 2)])
def test_spatial_axes(shape):
    from oracle import psn_oracle as O
    P = _P()
    rng = np.random.default_rng(16)
    x = rng.standard_normal(shape)
    w = rng.standard_normal((3, 2))
    b = rng.standard_normal(3)
    got = P.conv_forward(_t(x), _t(w), _t(b), d=2).cpu().numpy()
    assert np.array_equal(got, O.conv_forward(x, w, b, 2))
    dh = rng.standard_normal(shape)
    assert_close_scaled(P.conv_backward_weight(_t(x), _t(dh), 2, 2).cpu().numpy(),
                        O.conv_backward_weight(x, dh, 2, 2), 1e-12, "spatial bwd_w")


@pytest.mark.parametrize("shape,k,d,rows,dt", [((300, 7, 45), 4, 2, 45, torch.float32),
                                               ((64, 16, 128), 16, 3, 1, torch.float32),
                                               ((50, 4, 6, 3, 3), 3, 1, 6, torch.float64)])
def test_shift_spike_forward_is_the_two_step_composition(shape, k, d, rows, dt):
    """psn_shift_spike_forward (the quantized model layer in one pass) equals
    the reference's two steps, conv_forward_shift then (h >= 0), bit for bit,
    including exact-zero membranes (integer inputs)."""
    from paper_2501_14490_b200.engines import ShiftWeights, conv_forward_shift, shift_spike_forward
    g = torch.Generator().manual_seed(sum(shape) + k)
    sign = torch.randint(-1, 2, (rows, k), generator=g, dtype=torch.int8)
    expo = torch.randint(-3, 3, (rows, k), generator=g, dtype=torch.int8)
    sw = ShiftWeights(sign, expo)
    C = shape[2]
    bias = torch.randint(-2, 3, (C,), generator=g).double() * 0.5
    x = torch.randint(-3, 4, shape, generator=g).to(dt).cuda()
    two = (conv_forward_shift(x, sw, bias=bias, d=d) >= 0).to(dt)
    one = shift_spike_forward(x, sw, bias=bias, d=d)
    assert one.dtype == dt and torch.equal(one, two)
    xr = torch.randn(shape, generator=g).to(dt).cuda()
    assert torch.equal(shift_spike_forward(xr, sw, bias=bias, d=d), (conv_forward_shift(xr, sw, bias=bias, d=d) >= 0).to(dt))

"""CPU tests of the network container and the SSNN1 formats against fixtures
the reference itself wrote (tests/golden/make_golden_net.py): seeded
construction, byte-identical model / tensor round trips and format errors.
No CUDA compute (the model is built and (de)serialised on the CPU)."""

import os

import numpy as np
import pytest
import torch

from paper_2501_14490_b200 import modelio
from paper_2501_14490_b200.net import LinearLayer, ReadoutLayer, SpikingNet, build_task_net
from paper_2501_14490_b200.layer import ShiftLayer, SpikingLayer

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _z():
    return np.load(os.path.join(GOLDEN, "net_train.npz"))


def _net_cpu():
    T, N, IN, CH, CLASSES, ORDER, SEED = (int(v) for v in _z()["meta"])
    return build_task_net(channels=CH, num_layers=3, order=ORDER, classes=CLASSES, seed=SEED,
                          in_features=IN, device="cpu")


def test_seeded_build_reproduces_reference_weights():
    z = _z()
    net = _net_cpu()
    params = net.parameters_list()
    assert len(params) == sum(1 for k in z.files if k.startswith("init_"))
    for i, p in enumerate(params):
        assert np.array_equal(p.detach().numpy(), z[f"init_{i}"]), f"parameter {i}"
    kinds = [type(l).__name__ for l in net.layers]
    assert kinds == ["LinearLayer", "SpikingLayer"] * 3 + ["ReadoutLayer"]
    assert [l.cfg.dilation for l in net.spiking_layers()] == [1, 2, 3]


@pytest.mark.parametrize("name", ["ssnn1_float.bin", "ssnn1_quantized.bin"])
def test_model_file_round_trip_is_byte_identical(name, tmp_path):
    raw = open(os.path.join(GOLDEN, name), "rb").read()
    net, meta = modelio.model_from_bytes(raw, device="cpu")
    assert meta == {"version": 1, "quantized": name == "ssnn1_quantized.bin"}
    assert modelio.model_bytes(net) == raw
    p = str(tmp_path / "m.bin")
    modelio.save_model(net, p)
    net2, _ = modelio.load_model(p, device="cpu")
    assert modelio.model_bytes(net2) == raw
    want = (ShiftLayer if "quantized" in name else SpikingLayer)
    assert sum(isinstance(l, want) for l in net.layers) == 3
    assert isinstance(net.layers[0], LinearLayer) and isinstance(net.layers[-1], ReadoutLayer)


def test_float_model_file_carries_the_trained_parameters():
    """The reference's file of the trained net decodes to its f32-rounded
    parameters and running statistics (modelio.py:72-93)."""
    z = _z()
    net, _ = modelio.model_from_bytes(open(os.path.join(GOLDEN, "ssnn1_float.bin"), "rb").read(), device="cpu")
    for i, p in enumerate(net.parameters_list()):
        want = z[f"s1_after_{i}"].astype(np.float32).astype(np.float64)
        assert np.array_equal(p.detach().numpy(), want), f"parameter {i}"
    for j, l in enumerate(net.spiking_layers()):
        assert np.array_equal(l.running_mean.numpy(), z[f"s1_rm_{j}"].astype(np.float32).astype(np.float64))
        assert np.array_equal(l.running_var.numpy(), z[f"s1_rv_{j}"].astype(np.float32).astype(np.float64))
        assert l.eps == np.float32(1e-5) and l.momentum == np.float32(0.1)


def test_tensor_file_round_trip(tmp_path):
    raw = open(os.path.join(GOLDEN, "tensor_f32.bin"), "rb").read()
    t, layout = modelio.load_tensor(os.path.join(GOLDEN, "tensor_f32.bin"))
    assert layout == "time_first" and t.dtype == torch.float32 and tuple(t.shape) == (2, 3, 4)
    assert torch.equal(t, torch.arange(24, dtype=torch.float32).reshape(2, 3, 4) / 7)
    p = str(tmp_path / "t.bin")
    modelio.save_tensor(p, t, layout)
    assert open(p, "rb").read() == raw


def test_format_errors(tmp_path):
    raw = open(os.path.join(GOLDEN, "ssnn1_float.bin"), "rb").read()
    with pytest.raises(modelio.ModelFormatError, match="magic"):
        modelio.model_from_bytes(b"XXXXX" + raw[5:], device="cpu")
    with pytest.raises(modelio.ModelFormatError, match="truncated"):
        modelio.model_from_bytes(raw[:-3], device="cpu")
    with pytest.raises(modelio.ModelFormatError, match="trailing"):
        modelio.model_from_bytes(raw + b"\0", device="cpu")
    with pytest.raises(modelio.ModelFormatError, match="version"):
        modelio.model_from_bytes(raw[:5] + b"\x02\x00" + raw[7:], device="cpu")
    bad = bytearray(raw)
    bad[12] = 9  # first layer tag
    with pytest.raises(modelio.ModelFormatError, match="unknown layer tag"):
        modelio.model_from_bytes(bytes(bad), device="cpu")
    p = tmp_path / "t.bin"
    p.write_bytes(b"shiftsnn-tensor v1\ndtype=f32\nlayout=time_first\nshape=2,2\ndata\n" + b"\0" * 12)
    with pytest.raises(modelio.ModelFormatError, match="payload"):
        modelio.load_tensor(str(p))
    p.write_bytes(b"nope")
    with pytest.raises(modelio.ModelFormatError):
        modelio.load_tensor(str(p))
    with pytest.raises(ValueError):
        SpikingNet([])
    with pytest.raises(ValueError):
        ReadoutLayer(4, 2, tau=1.0, device="cpu")

"""Golden fixtures for the network around the neuron (SURVEY.md section 8(f)
ranks 2-3): the reference's SpikingNet training step with Adam, and its SSNN1
model / tensor files.

Run IN THE BUILD CONTAINER ONLY (imports the read-only reference from
/root/reference/pkg/src, absent on the GPU box):

    python tests/golden/make_golden_net.py

Writes tests/golden/net_train.npz, tests/golden/ssnn1_float.bin,
tests/golden/ssnn1_quantized.bin, tests/golden/tensor_f32.bin.

The network is the reference's build_task_net (train.py:105-135) with an
input synapse of IN features instead of 1 (SHD-shaped inputs feed 700); it is
assembled here with exactly build_task_net's RNG call sequence, which
paper_2501_14490_b200.net.build_task_net(in_features=IN) reproduces.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

T, N, IN, CH, CLASSES, ORDER, SEED = 20, 6, 12, 8, 4, 3, 5
LR = 1e-2


def build_ref_net(ref, in_features):
    network, neuron, surrogate, tensor = ref
    dilations = neuron.sawtooth_schedule(3)
    rng = np.random.default_rng(SEED)
    sur = surrogate.SurrogateConfig()
    layers, prev = [], in_features
    for d in dilations:  # train.py:124-134 with prev = in_features
        layers.append(network.LinearLayer(prev, CH, rng=rng))
        cfg = neuron.NeuronConfig(channels=CH, order=ORDER, dilation=d, quantized=True)
        layers.append(network.SpikingLayer(cfg, surrogate=sur, weight_init="uniform", rng=rng))
        prev = CH
    layers.append(network.ReadoutLayer(CH, CLASSES, rng=rng))
    return network.SpikingNet(layers, tensor.Layout.TIME_FIRST)


def main():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import importlib
    from shiftsnn import modelio, network, neuron, surrogate, tensor
    train = importlib.import_module("shiftsnn.train")  # the package re-exports a function `train`
    ref = (network, neuron, surrogate, tensor)
    net = build_ref_net(ref, IN)
    out = {"meta": np.array([T, N, IN, CH, CLASSES, ORDER, SEED]), "lr": np.array(LR)}
    params = net.parameters()
    for i, p in enumerate(params):
        out[f"init_{i}"] = p.value.copy()
    rng = np.random.default_rng(77)
    xs, ys = [], []
    opt = train.Adam(LR)
    for step in range(2):
        x = (rng.random((T, N, IN)) < 0.3).astype(np.float64)  # spike-train input
        y = rng.integers(0, CLASSES, N)
        xs.append(x)
        ys.append(y)
        loss, acc = net.train_step_grads(tensor.TemporalTensor(x, tensor.Layout.TIME_FIRST), y)
        out[f"s{step}_x"], out[f"s{step}_y"] = x, y
        out[f"s{step}_loss"], out[f"s{step}_acc"] = np.array(loss), np.array(acc)
        for i, p in enumerate(params):
            out[f"s{step}_grad_{i}"] = p.grad.copy()
        for j, layer in enumerate(net.spiking_layers()):
            out[f"s{step}_rm_{j}"] = layer.thr.running_mean.copy()
            out[f"s{step}_rv_{j}"] = layer.thr.running_var.copy()
        opt.step(params)
        for i, p in enumerate(params):
            out[f"s{step}_after_{i}"] = p.value.copy()
    xe = (rng.random((T, N, IN)) < 0.3).astype(np.float64)
    out["eval_x"] = xe
    out["eval_logits"] = np.asarray(net.forward(tensor.TemporalTensor(xe, tensor.Layout.TIME_FIRST),
                                                network.Mode.EVAL))
    out["eval_pred"] = net.predict(tensor.TemporalTensor(xe, tensor.Layout.TIME_FIRST))
    np.savez_compressed(os.path.join(HERE, "net_train.npz"), **out)

    modelio.save_model(net, os.path.join(HERE, "ssnn1_float.bin"), quantize=False)
    modelio.save_model(net, os.path.join(HERE, "ssnn1_quantized.bin"), quantize=True)
    # the quantized file reloads as ShiftLayers; its EVAL logits on xe
    qnet, _ = modelio.load_model(os.path.join(HERE, "ssnn1_quantized.bin"))
    out2 = {"q_eval_logits": np.asarray(qnet.forward(tensor.TemporalTensor(xe, tensor.Layout.TIME_FIRST),
                                                     network.Mode.EVAL))}
    np.savez_compressed(os.path.join(HERE, "net_quantized_eval.npz"), **out2)
    t = tensor.TemporalTensor(np.arange(2 * 3 * 4, dtype=np.float32).reshape(2, 3, 4) / 7,
                              tensor.Layout.TIME_FIRST)
    modelio.save_tensor(os.path.join(HERE, "tensor_f32.bin"), t)
    print("wrote net_train.npz, net_quantized_eval.npz, ssnn1_float.bin, ssnn1_quantized.bin, tensor_f32.bin")


if __name__ == "__main__":
    main()

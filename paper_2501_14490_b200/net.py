"""The network around the neuron: the reference's ``SpikingNet`` training step
 on the GPU.

* ``LinearLayer``   stateless synapse, network.py:80-140 (cuBLAS GEMM: a plain
                    library GEMM, as the north star allows for the synapses)
* ``ReadoutLayer``  leaky accumulator readout, network.py:365-436, run as a
                    weighted time reduction by the CUDA kernels
                    ``psn_readout_reduce`` / ``psn_readout_expand``
* ``ce_loss``       cross entropy, network.py:67-77
* ``SpikingNet``    the layer stack, network.py:439-496
                    (``train_step_grads``, ``loss``, ``predict``)
* ``SGD`` / ``Adam``  train.py:138-172, element for element the reference's update
* ``build_task_net``  train.py:105-135 (same seeded RNG call sequence, so a
                    seeded build reproduces the reference's weights), with an
                    ``in_features`` argument for SHD-shaped inputs (700)

Parameters are float64 like the reference's.  The carrier dtype of the
activations is the dtype of the input: float64 reproduces the reference's
TRAIN arithmetic; float32 / bfloat16 run the neuron layers on the streamed
sm_100a kernels (the production setting, BASELINE configs[1]).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.nn.functional as F
from torch import nn

from . import _lib as L
from .layer import Mode, ShiftLayer, SpikingLayer
from .neuron import NeuronConfig, QuantGradMode, SurrogateConfig, WeightSharing, sawtooth_schedule


class _LinearF32(torch.autograd.Function):
    """The synapse on an f32 carrier with a backward shaped for its long
    reduction (T*N rows, a few hundred columns): the weight gradient as a
    split-K batched GEMM (S slices of the rows, partial products summed in a
    fixed order), the bias gradient as a ones-vector GEMV.  cuBLAS's single
    GEMM for dW = dy^T x puts one 128x128 output tile on a handful of SMs
    (SHD shape: 107 -> 36 us for 128x128, 223 -> 120 us for 128x700;
    scripts/mb_linear_bwd.py)."""

    @staticmethod
    def forward(ctx, x, W, b):
        W32 = W.to(x.dtype)
        ctx.save_for_backward(x, W32)
        return F.linear(x, W32, b.to(x.dtype))

    @staticmethod
    def backward(ctx, gy):
        x, W32 = ctx.saved_tensors
        out_f, in_f = W32.shape
        R = x.numel() // in_f
        g2 = gy.reshape(R, out_f)
        x2 = x.reshape(R, in_f)
        dx = (g2 @ W32).reshape(x.shape) if ctx.needs_input_grad[0] else None
        S = next((s for s in (32, 16, 8, 4, 2) if R % s == 0 and R // s >= 256), 1)
        if S > 1:
            dW = torch.bmm(g2.view(S, R // S, out_f).transpose(1, 2), x2.view(S, R // S, in_f)).sum(0)
        else:
            dW = g2.t() @ x2
        db = (torch.ones((1, R), dtype=g2.dtype, device=g2.device) @ g2).view(out_f)
        return dx, dW.to(torch.float64), db.to(torch.float64)


class LinearLayer(nn.Module):
    """One weight matrix shared across all time steps (network.py:80-140);
    rank-3 time-first inputs [T, N, in] -> [T, N, out].  f32 CUDA carriers
    take the split-K weight-gradient backward (_LinearF32)."""

    def __init__(self, in_features: int, out_features: int, rng: np.random.Generator | None = None,
                 *, device=None):
        super().__init__()
        rng = rng or np.random.default_rng()
        w = rng.normal(0.0, in_features ** -0.5, size=(out_features, in_features))
        dev = _device(device)
        self.W = nn.Parameter(torch.tensor(w, dtype=torch.float64, device=dev))
        self.b = nn.Parameter(torch.zeros(out_features, dtype=torch.float64, device=dev))

    def out_channels(self) -> int:
        return self.W.shape[0]

    def forward(self, x: torch.Tensor, mode: Mode = Mode.TRAIN) -> torch.Tensor:
        if x.dim() != 3:
            raise ValueError("linear layers take rank-3 tensors")
        if mode is Mode.EVAL:  # deployment path in f32 (network.py:113-116)
            return F.linear(x.to(torch.float32), self.W.to(torch.float32), self.b.to(torch.float32))
        if x.is_cuda and x.dtype == torch.float32:
            return _LinearF32.apply(x.contiguous(), self.W, self.b)
        return F.linear(x, self.W.to(x.dtype), self.b.to(x.dtype))


class _ReadoutReduce(torch.autograd.Function):
    """xbar[n, c] = sum_t w_t x[t, n, c] (f64) and its broadcast backward."""

    @staticmethod
    def forward(ctx, x, tau):
        T, N, C = x.shape
        x = x.contiguous()
        xbar = torch.empty((N, C), dtype=torch.float64, device=x.device)
        L.run(x, "psn_readout_reduce", T, N, C, L.dtype_code(x.dtype), float(tau), L.ptr(x), L.ptr(xbar),
              L.stream_of(x))
        ctx.meta = (T, N, C, x.dtype, float(tau))
        return xbar

    @staticmethod
    def backward(ctx, gbar):
        T, N, C, dt, tau = ctx.meta
        g = gbar.to(torch.float64).contiguous()
        dx = torch.empty((T, N, C), dtype=dt, device=g.device)
        L.run(g, "psn_readout_expand", T, N, C, L.dtype_code(dt), tau, L.ptr(g), L.ptr(dx), L.stream_of(g))
        return dx, None


class ReadoutLayer(nn.Module):
    """Non-spiking leaky accumulator readout (network.py:365-436): the class
    scores are the membrane potentials after the last step,
    v_T = sum_t (1/tau)(1 - 1/tau)^(T-1-t) (x[t] W^T + b)."""

    def __init__(self, in_features: int, classes: int, tau: float = 2.0,
                 rng: np.random.Generator | None = None, *, device=None):
        super().__init__()
        if tau <= 1:
            raise ValueError("tau must be > 1")
        rng = rng or np.random.default_rng()
        w = rng.normal(0.0, in_features ** -0.5, size=(classes, in_features))
        dev = _device(device)
        self.W = nn.Parameter(torch.tensor(w, dtype=torch.float64, device=dev))
        self.b = nn.Parameter(torch.zeros(classes, dtype=torch.float64, device=dev))
        self.tau = float(tau)

    def out_channels(self) -> int:
        return self.W.shape[0]

    def forward(self, x: torch.Tensor, mode: Mode = Mode.TRAIN) -> torch.Tensor:
        if x.dim() != 3:
            raise ValueError("readout takes rank-3 tensors")
        L.require_cuda(x)
        keep = 1.0 - 1.0 / self.tau
        wsum = 1.0 - keep ** x.shape[0]  # sum_t w_t
        if mode is Mode.EVAL:  # f32 deployment path (network.py:401-405)
            xbar = _ReadoutReduce.apply(x.to(torch.float32), self.tau).to(torch.float32)
            return F.linear(xbar, self.W.to(torch.float32)) + self.b.to(torch.float32) * float(wsum)
        xbar = _ReadoutReduce.apply(x, self.tau)
        return F.linear(xbar, self.W) + self.b * wsum


def ce_loss(logits: torch.Tensor, labels: torch.Tensor):
    """Cross entropy (network.py:67-77): mean over the batch; returns (loss,
    accuracy) tensors, the gradient by autograd is (softmax - onehot) / n."""
    n = logits.shape[0]
    z = logits - logits.max(dim=1, keepdim=True).values.detach()
    lse = torch.log(torch.exp(z).sum(dim=1))
    loss = torch.mean(lse - z[torch.arange(n, device=logits.device), labels])
    acc = (torch.argmax(logits.detach(), dim=1) == labels).to(torch.float64).mean()
    return loss, acc


class SpikingNet(nn.Module):
    """A stack of layers ending in a readout (network.py:439-496)."""

    def __init__(self, layers: list):
        super().__init__()
        if not layers:
            raise ValueError("network must have at least one layer")
        self.layers = nn.ModuleList(layers)

    def spiking_layers(self) -> list:
        return [l for l in self.layers if isinstance(l, SpikingLayer)]

    def parameters_list(self) -> list:
        """Parameters in the reference's order (per layer: W, b / W, gamma, beta)."""
        out = []
        for layer in self.layers:
            if isinstance(layer, SpikingLayer):
                out += [layer.W, layer.gamma, layer.beta]
            elif isinstance(layer, (LinearLayer, ReadoutLayer)):
                out += [layer.W, layer.b]
        return out

    def zero_grad(self, set_to_none: bool = False) -> None:
        live = []
        for p in self.parameters_list():
            if set_to_none or p.grad is None:
                p.grad = None if set_to_none else torch.zeros_like(p)
            else:
                live.append(p.grad)
        if live:
            torch._foreach_zero_(live)  # one multi-tensor launch instead of one fill per parameter

    def forward(self, x: torch.Tensor, mode: Mode = Mode.TRAIN) -> torch.Tensor:
        h = x
        for layer in self.layers:
            h = layer(h, mode)
        self._last_out = h if mode is not Mode.EVAL else None
        return h

    def backward(self, dlogits: torch.Tensor):
        """Explicit backward of the last TRAIN / SMOOTH forward from the logits'
        gradient (network.py:474-478); gradients accumulate into .grad."""
        out = getattr(self, "_last_out", None)
        if out is None:
            raise RuntimeError("backward() before a TRAIN / SMOOTH forward")
        out.backward(torch.as_tensor(dlogits, dtype=out.dtype, device=out.device))
        self._last_out = None

    def loss(self, x: torch.Tensor, labels: torch.Tensor, mode: Mode = Mode.TRAIN):
        """Forward + cross entropy; returns (loss, accuracy) tensors."""
        return ce_loss(self.forward(x, mode).to(torch.float64), labels)

    def train_step_grads_async(self, x: torch.Tensor, labels: torch.Tensor, mode: Mode = Mode.TRAIN):
        """train_step_grads without the host synchronisation: (loss, acc) tensors."""
        self.zero_grad()
        loss, acc = self.loss(x, labels, mode)
        loss.backward()
        self._last_out = None  # release the autograd graph (and its AccumulateGrad nodes' stream)
        return loss.detach(), acc

    def train_step_grads(self, x: torch.Tensor, labels: torch.Tensor, mode: Mode = Mode.TRAIN):
        """zero_grad, forward, cross entropy, backward (network.py:485-491);
        gradients land in .grad; returns (loss, accuracy) as floats."""
        loss, acc = self.train_step_grads_async(x, labels, mode)
        return float(loss), float(acc)

    @torch.no_grad()
    def predict(self, x: torch.Tensor) -> torch.Tensor:
        return torch.argmax(self.forward(x, Mode.EVAL), dim=1)


class SGD:
    """p -= lr * grad (train.py:138-144)."""

    def __init__(self, params, lr: float):
        self.params = list(params)
        self.lr = lr

    @torch.no_grad()
    def step(self) -> None:
        for p in self.params:
            p.sub_(self.lr * p.grad)


class Adam:
    """The reference's Adam (train.py:147-172), the same element-wise
    operations in the same order, so the update is bit-identical for the same
    gradients (IEEE f64 element-wise arithmetic).  CUDA float64 parameters
    are updated by one launch for all tensors (psn_adam_step over a device
    table of 4096-element chunks); CPU parameters by the element-wise torch
    formulation."""

    CHUNK = 4096

    def __init__(self, params, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8):
        self.params = list(params)
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.t = 0
        self._state = {}
        self._t_dev = None  # capturable mode: the step count lives on the device
        self._table, self._table_key = None, None

    def _fused_ok(self) -> bool:
        return all(p.is_cuda and p.dtype == torch.float64 and p.is_contiguous() and p.grad is not None
                   and p.grad.dtype == torch.float64 and p.grad.is_contiguous() for p in self.params)

    def _chunk_table(self) -> torch.Tensor:
        """Device table of (param, grad, m, v, n) chunks; rebuilt only when a
        tensor moved (never inside a captured step once warmed up)."""
        for p in self.params:
            if id(p) not in self._state:
                self._state[id(p)] = (torch.zeros_like(p), torch.zeros_like(p))
        key = tuple((p.data_ptr(), p.grad.data_ptr()) for p in self.params)
        if key != self._table_key:
            rows = []
            for p in self.params:
                m, v = self._state[id(p)]
                base = (p.data_ptr(), p.grad.data_ptr(), m.data_ptr(), v.data_ptr())
                for off in range(0, p.numel(), self.CHUNK):
                    rows.append([b + 8 * off for b in base] + [min(self.CHUNK, p.numel() - off)])
            self._table = torch.tensor(rows, dtype=torch.int64, device=self.params[0].device)
            self._table_key = key
        return self._table

    def make_capturable(self) -> None:
        """Keep the step count on the device so a captured step (CUDA graph)
        advances the bias corrections on every replay; the corrections are then
        1 - beta^t from the device pow (within an ulp of the host's)."""
        if self._t_dev is None:
            self._t_dev = torch.full((), float(self.t), dtype=torch.float64, device=self.params[0].device)

    @torch.no_grad()
    def step(self) -> None:
        self.t += 1
        b1, b2 = self.beta1, self.beta2
        dev_t = self._t_dev is not None
        if dev_t:
            self._t_dev.add_(1.0)
        if self.params and self._fused_ok():
            tab = self._chunk_table()
            p0 = self.params[0]
            c1h, c2h = (0.0, 0.0) if dev_t else (1 - b1 ** self.t, 1 - b2 ** self.t)
            L.run(p0, "psn_adam_step", L.ptr(tab), tab.shape[0], float(self.lr), float(b1), float(b2),
                  float(self.eps), float(c1h), float(c2h), L.ptr(self._t_dev) if dev_t else None, L.stream_of(p0))
            return
        if dev_t:
            c1 = 1 - torch.pow(b1, self._t_dev)
            c2 = 1 - torch.pow(b2, self._t_dev)
        else:
            c1, c2 = 1 - b1 ** self.t, 1 - b2 ** self.t
        for p in self.params:
            st = self._state.get(id(p))
            if st is None:
                st = self._state[id(p)] = (torch.zeros_like(p), torch.zeros_like(p))
            m, v = st
            g = p.grad
            m.mul_(b1)
            m.add_((1 - b1) * g)
            v.mul_(b2)
            v.add_((1 - b2) * g * g)
            mh = m / c1
            vh = v / c2
            p.sub_(self.lr * mh / (torch.sqrt(vh) + self.eps))


class GraphedTrainStep:
    """One training step (zero_grad, forward, cross entropy, backward,
    optimizer update) captured into a CUDA graph and replayed on static
    input / label buffers: the step is then one graph launch instead of a few
    hundred small kernel launches (the C-ABI calls are stream-ordered and
    allocation-free, so they capture).  Use: ``step = GraphedTrainStep(net,
    opt, x, y)``; copy the next batch into ``step.x`` / ``step.y``;
    ``loss, acc = step()`` (device tensors, no host synchronisation)."""

    def __init__(self, net: SpikingNet, opt, x: torch.Tensor, labels: torch.Tensor, warmup: int = 3):
        self.net, self.opt = net, opt
        if hasattr(opt, "make_capturable"):
            opt.make_capturable()
        self.x, self.y = x.clone(), labels.clone()
        side = torch.cuda.Stream(x.device)
        side.wait_stream(torch.cuda.current_stream(x.device))
        with torch.cuda.stream(side):  # warm-up (workspaces, grads, optimizer state) off the capture
            for _ in range(warmup):
                net.train_step_grads_async(self.x, self.y)
                opt.step()
        torch.cuda.current_stream(x.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss, self.acc = net.train_step_grads_async(self.x, self.y)
            opt.step()

    def __call__(self):
        self.graph.replay()
        return self.loss, self.acc


def build_task_net(channels: int = 24, num_layers: int = 3, order: int = 2,
                   dilations: list | None = None, classes: int = 2, quantized: bool = True,
                   grad_mode: QuantGradMode = QuantGradMode.WHOLE_STE,
                   weight_sharing: WeightSharing = WeightSharing.CHANNEL_WISE,
                   surrogate: SurrogateConfig | None = None, seed: int = 0,
                   in_features: int = 1, *, device=None) -> SpikingNet:
    """Input synapse, a stack of (synapse, spiking layer) blocks with sawtooth
    dilations, and a class readout (train.py:105-135).  ``in_features`` is 1
    in the reference's toy tasks; 700 for SHD-shaped inputs."""
    if dilations is None:
        dilations = sawtooth_schedule(num_layers)
    if len(dilations) != num_layers:
        raise ValueError("need one dilation per layer")
    rng = np.random.default_rng(seed)
    surrogate = surrogate or SurrogateConfig()
    layers: list = []
    prev = in_features
    for d in dilations:
        layers.append(LinearLayer(prev, channels, rng=rng, device=device))
        cfg = NeuronConfig(channels=channels, order=order, dilation=d, weight_sharing=weight_sharing,
                           quantized=quantized, grad_mode=grad_mode)
        layers.append(SpikingLayer(cfg, surrogate=surrogate, weight_init="uniform", rng=rng, device=device))
        prev = channels
    layers.append(ReadoutLayer(channels, classes, rng=rng, device=device))
    return SpikingNet(layers)


def _device(device):
    if device is not None:
        return torch.device(device)
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


__all__ = ["LinearLayer", "ReadoutLayer", "ShiftLayer", "SpikingNet", "ce_loss", "SGD", "Adam",
           "GraphedTrainStep", "build_task_net"]

"""SpikingLayer — the reference's neuron module (src/network.py:143-318) as a
torch ``nn.Module`` whose forward and backward are the sm_100a kernels of
libpsn_b200.so, reached through the C ABI by a ``torch.autograd.Function``.

Constructor, modes and semantics follow the reference:

* ``SpikingLayer(cfg, surrogate=None, weight_init="lif", rng=None,
  fuse_from_batch_stats=True)`` (network.py:146-160); parameters ``W``
  (C, k) or shared (1, k), ``gamma`` = 1, ``beta`` = -1, buffers
  ``running_mean`` = 0 / ``running_var`` = 1, ``eps`` 1e-5, ``momentum`` 0.1,
  all float64 like the reference's.
* ``forward(x, mode)`` with ``Mode.TRAIN`` (batch statistics, running update,
  quantization-aware double pass, Heaviside spikes), ``Mode.SMOOTH``
  (spike primitive, statistics frozen) or ``Mode.EVAL`` (running statistics
  folded, pow2 shift execution).  ``mode=None`` follows ``self.training``.
* gradients flow by autograd into ``W.grad``, ``gamma.grad``, ``beta.grad``
  (accumulating, as the reference's ``+=``) and into ``x``.

``x`` is a time-first CUDA tensor ``[T, N, C]`` or ``[T, N, C, H(, W)]`` of
dtype float32, bfloat16 or float64; outputs have the dtype of ``x``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch
from torch import nn

from . import _lib as L
from .engines import ShiftWeights, shift_spike_forward
from .neuron import (BN_EPS_DEFAULT, BN_MOMENTUM_DEFAULT, NeuronConfig, QuantGradMode,
                     SurrogateConfig, SurrogateKind, WeightSharing, init_weights)


class Mode(Enum):
    TRAIN = "train"
    SMOOTH = "smooth"
    EVAL = "eval"


@dataclass(frozen=True)
class LayerMethod:
    """One implementation choice of a layer (network.py:58-64): "auto" lets
    the planner pick the streamed persistent kernels or the generic
    three-launch kernels from the shape (small or widest-window shapes take
    the generic ones); "stream" takes the streamed kernels whenever the shape
    allows (descriptor flag PSN_STREAM); "generic" always takes the
    three-launch kernels (PSN_GENERIC).  The reference's engine registry is a
    CPU stand-in for GPU methods, out of scope."""

    name: str = "auto"
    engine: object = None
    block_size: int | None = None


def _surrogate_code(s: SurrogateConfig) -> int:
    return L.PSN_ARCTAN if s.kind is SurrogateKind.ARCTAN else L.PSN_RATIONAL


class _PSNFunction(torch.autograd.Function):
    """One TRAIN/SMOOTH forward + its backward through the C ABI."""

    @staticmethod
    def forward(ctx, x, W, gamma, beta, running_mean, running_var, desc_args, layer):
        desc = L.make_desc(x.shape, *desc_args)
        out = torch.empty_like(x)
        fold = torch.empty((x.shape[2], L.fold_stride(desc.k)), dtype=torch.float64, device=x.device)
        ws = L.workspace_for(desc, x.device, L.stream_of(x))
        L.run(x, "psn_forward_train", ctypes.byref(desc), L.ptr(x), L.ptr(W), L.ptr(gamma), L.ptr(beta),
                                      L.ptr(running_mean), L.ptr(running_var), L.ptr(out), L.ptr(fold),
                                      L.ptr(ws), L.stream_of(x))
        ctx.save_for_backward(x, W, gamma, fold)
        ctx.desc_args = desc_args
        if layer is not None:
            layer.last_fold = fold
            layer._last = (x.detach(), desc_args)  # what the explicit backward(dy) consumes
        return out

    @staticmethod
    def backward(ctx, dy):
        x, W, gamma, fold = ctx.saved_tensors
        desc = L.make_desc(x.shape, *ctx.desc_args)
        dy = dy.to(x.dtype).contiguous()
        dx = torch.empty_like(x)
        dW = torch.empty_like(W)
        dgamma = torch.empty_like(gamma)
        dbeta = torch.empty_like(gamma)
        ws = L.workspace_for(desc, x.device, L.stream_of(x))
        L.run(x, "psn_backward", ctypes.byref(desc), L.ptr(x), L.ptr(dy), L.ptr(W), L.ptr(gamma),
                                     L.ptr(fold), L.ptr(dx), L.ptr(dW), L.ptr(dgamma), L.ptr(dbeta),
                                     L.ptr(ws), L.stream_of(x))
        return dx, dW, dgamma, dbeta, None, None, None, None


class SpikingLayer(nn.Module):
    """Channel-wise mul-free parallel spiking neuron with a BN threshold."""

    def __init__(self, cfg: NeuronConfig, surrogate: SurrogateConfig | None = None,
                 weight_init: str = "lif", rng: np.random.Generator | None = None,
                 fuse_from_batch_stats: bool = True, *, device=None):
        super().__init__()
        if cfg.order > L.PSN_MAX_ORDER_PY:
            raise ValueError(f"order {cfg.order} above the kernel limit {L.PSN_MAX_ORDER_PY}")
        self.cfg = cfg
        self.surrogate = surrogate or SurrogateConfig()
        dev = torch.device(device) if device is not None else (
            torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
        W = init_weights(cfg, kind=weight_init, rng=rng)
        C = cfg.channels
        self.W = nn.Parameter(torch.tensor(W, dtype=torch.float64, device=dev))
        self.gamma = nn.Parameter(torch.ones(C, dtype=torch.float64, device=dev))
        self.beta = nn.Parameter(-torch.ones(C, dtype=torch.float64, device=dev))
        self.register_buffer("running_mean", torch.zeros(C, dtype=torch.float64, device=dev))
        self.register_buffer("running_var", torch.ones(C, dtype=torch.float64, device=dev))
        self.eps = BN_EPS_DEFAULT
        self.momentum = BN_MOMENTUM_DEFAULT
        self.fuse_from_batch_stats = fuse_from_batch_stats
        self.quantize_in_smooth_mode = False
        self.last_fold = None
        self._last = None
        self.method = LayerMethod("auto")

    # -- reference-compatible helpers (network.py:162-209) ----------------------
    def out_channels(self) -> int:
        return self.cfg.channels

    def parameters_list(self) -> list:
        """[W, gamma, beta], the reference's parameters() order."""
        return [self.W, self.gamma, self.beta]

    def method_candidates(self, layout=None) -> list:
        return [LayerMethod("auto"), LayerMethod("stream"), LayerMethod("generic")]

    def configure(self, method: LayerMethod) -> None:
        if method.name not in ("auto", "stream", "generic"):
            raise ValueError(f"unknown layer method {method.name!r} ('auto', 'stream' or 'generic')")
        self.method = method

    def backward(self, dy: torch.Tensor) -> torch.Tensor:
        """Explicit backward of the last TRAIN / SMOOTH forward, as the
        reference's SpikingLayer.backward(dy) (network.py:272-318): gradients
        ACCUMULATE into W.grad, gamma.grad, beta.grad; returns dx (dtype of x).
        (Autograd through forward() is the usual route; this one serves code
        written against the reference's layer-by-layer backward.)"""
        if getattr(self, "_last", None) is None or self.last_fold is None:
            raise RuntimeError("backward() before a TRAIN / SMOOTH forward")
        x, desc_args = self._last
        desc = L.make_desc(x.shape, *desc_args)
        dy = dy.to(x.dtype).contiguous()
        if tuple(dy.shape) != tuple(x.shape):
            raise ValueError(f"dy has shape {tuple(dy.shape)}, the forward's input {tuple(x.shape)}")
        dx = torch.empty_like(x)
        dW, dg, db = torch.empty_like(self.W), torch.empty_like(self.gamma), torch.empty_like(self.gamma)
        ws = L.workspace_for(desc, x.device, L.stream_of(x))
        L.run(x, "psn_backward", ctypes.byref(desc), L.ptr(x), L.ptr(dy), L.ptr(self.W), L.ptr(self.gamma),
              L.ptr(self.last_fold), L.ptr(dx), L.ptr(dW), L.ptr(dg), L.ptr(db), L.ptr(ws), L.stream_of(x))
        with torch.no_grad():
            for p, g in ((self.W, dW), (self.gamma, dg), (self.beta, db)):
                if p.grad is None:
                    p.grad = g
                else:
                    p.grad.add_(g)
        return dx

    def _flags(self, mode: Mode) -> int:
        f = 0
        if self.cfg.quantized:
            f |= L.PSN_QUANTIZED
        if self.cfg.weight_sharing is WeightSharing.SHARED:
            f |= L.PSN_SHARED
        if self.fuse_from_batch_stats:
            f |= L.PSN_USE_BATCH_STATS
        if mode is Mode.SMOOTH:
            f |= L.PSN_SMOOTH
        if self.quantize_in_smooth_mode:
            f |= L.PSN_QUANTIZE_IN_SMOOTH
        if self.cfg.grad_mode is QuantGradMode.ROUND_STE:
            f |= L.PSN_ROUND_STE
        if self.method.name == "generic":
            f |= L.PSN_GENERIC
        elif self.method.name == "stream":
            f |= L.PSN_STREAM
        return f

    def _desc_args(self, mode: Mode):
        return (self.cfg.order, self.cfg.dilation, None, self._flags(mode),
                _surrogate_code(self.surrogate), self.surrogate.alpha, self.eps, self.momentum)

    def _check_input(self, x: torch.Tensor) -> torch.Tensor:
        L.require_cuda(x)
        if not 3 <= x.dim() <= 5:
            raise ValueError(f"rank must be 3..5 (T, N, C plus up to 2 spatial axes), got {x.dim()}")
        if x.shape[2] != self.cfg.channels:
            raise ValueError(f"input has {x.shape[2]} channels, config expects {self.cfg.channels}")
        if x.dtype not in (torch.float32, torch.bfloat16, torch.float64):
            # the reference's TemporalTensor converts any other dtype to float64
            # (tensor.py:17, 57-59), and its outputs then carry float64 too
            x = x.to(torch.float64)
        return x.contiguous()

    def fused_running(self):
        """Running statistics folded into (W_f, b_f) (neuron.py:228-244)."""
        scale = self.gamma.detach() / torch.sqrt(self.running_var + self.eps)
        W = self.W.detach()
        if W.shape[0] == 1 and self.cfg.channels > 1:
            W = W.expand(self.cfg.channels, W.shape[1])
        return W * scale[:, None], self.beta.detach() - scale * self.running_mean

    def quantized_snapshot(self):
        """(ShiftWeights, f32 bias) a quantized model file carries (network.py:207-209)."""
        from .engines import quantize_pow2
        w_f, b_f = self.fused_running()
        return quantize_pow2(w_f), b_f.to(torch.float32)

    # -- forward ----------------------------------------------------------------
    def forward(self, x: torch.Tensor, mode: Mode | None = None) -> torch.Tensor:
        if mode is None:
            mode = Mode.TRAIN if self.training else Mode.EVAL
        x = self._check_input(x)
        args = list(self._desc_args(mode))
        args[2] = x.dtype
        if mode is Mode.EVAL:
            return self._forward_eval(x, tuple(args))
        return _PSNFunction.apply(x, self.W, self.gamma, self.beta, self.running_mean,
                                  self.running_var, tuple(args), self)

    def _forward_eval(self, x, args) -> torch.Tensor:
        desc = L.make_desc(x.shape, *args)
        out = torch.empty_like(x)
        ws = L.workspace(desc, x.device)
        with torch.no_grad():
            L.run(x, "psn_forward_eval", ctypes.byref(desc), L.ptr(x), L.ptr(self.W), L.ptr(self.gamma),
                                             L.ptr(self.beta), L.ptr(self.running_mean),
                                             L.ptr(self.running_var), L.ptr(out), L.ptr(ws), L.stream_of(x))
        return out

    # -- inspection of the last TRAIN/SMOOTH forward (the reference's _cache) ---
    def last_state(self) -> dict:
        """mu*, s, a, b_f, batch mean/var, w_f, w_q of the last forward, and (streamed
        forward) the BN-term data sums sx, cx the backward's dW uses."""
        f = self.last_fold
        if f is None:
            raise RuntimeError("no forward has run yet")
        k = self.cfg.order
        return {"mu": f[:, 0], "s": f[:, 1], "a": f[:, 2], "b_f": f[:, 3],
                "mu_batch": f[:, 4], "var_batch": f[:, 5],
                "w_f": f[:, L.PSN_FOLD_HDR:L.PSN_FOLD_HDR + k],
                "w_q": f[:, L.PSN_FOLD_HDR + k:L.PSN_FOLD_HDR + 2 * k],
                "sx": f[:, L.PSN_FOLD_HDR + 2 * k:L.PSN_FOLD_HDR + 3 * k],
                "cx": f[:, L.PSN_FOLD_HDR + 3 * k:L.PSN_FOLD_HDR + 4 * k]}


class ShiftLayer(nn.Module):
    """Inference-only layer of fused pow2 weights plus an f32 bias
    (src/network.py:321-362): what a quantized model deserialises to."""

    def __init__(self, sw: ShiftWeights, bias_f32, dilation: int):
        super().__init__()
        if sw.sign.dim() != 2:
            raise ValueError("shift weights must be (C, k)")
        bias = torch.as_tensor(bias_f32, dtype=torch.float32)
        if tuple(bias.shape) != (sw.shape[0],):
            raise ValueError("bias must have one entry per channel")
        self.sw = sw
        self.register_buffer("bias", bias)
        self.dilation = dilation

    def out_channels(self) -> int:
        return self.sw.shape[0]

    def forward(self, x: torch.Tensor, mode: Mode = Mode.EVAL) -> torch.Tensor:
        if mode is not Mode.EVAL:
            raise ValueError("quantized fused layers are inference-only")
        L.require_cuda(x)
        x32 = x.to(torch.float32).contiguous()
        return shift_spike_forward(x32, self.sw, bias=self.bias.to(x32.device, torch.float64), d=self.dilation)

    def backward(self, dy):
        raise ValueError("quantized fused layers are inference-only")

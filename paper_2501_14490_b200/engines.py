"""Engine-level operators on the GPU — the reference's operator ("plugin")
API for the path, one fused CUDA family instead of a CPU engine registry.

Mirrors src/engines.py:336-431 and src/quant.py:54-144: same function names,
argument meaning and errors.  Tensors are time-first ``[T, N, C, *spatial]``
CUDA tensors; weights are ``(C, k)`` or shared ``(1, k)`` float64.  The
forward / shift / backward-input convolutions accumulate in float64 in the
reference's tap order and are bit-identical to its DIRECT engine.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib as L
from .neuron import E_MAX, E_MIN


@dataclass
class ShiftWeights:
    """Quantized weights sign * 2**exponent (src/quant.py:54-80); int8 tensors."""

    sign: torch.Tensor
    exponent: torch.Tensor

    def __post_init__(self):
        self.sign = torch.as_tensor(self.sign).to(torch.int8)
        self.exponent = torch.as_tensor(self.exponent).to(torch.int8)
        if self.sign.shape != self.exponent.shape:
            raise ValueError("sign and exponent shapes differ")
        if not bool(torch.isin(self.sign, torch.tensor([-1, 0, 1], dtype=torch.int8,
                                                        device=self.sign.device)).all()):
            raise ValueError("sign values must be in {-1, 0, +1}")
        if bool(((self.exponent < E_MIN) | (self.exponent > E_MAX)).any()):
            raise ValueError(f"exponent out of [{E_MIN}, {E_MAX}]")

    @property
    def shape(self):
        return tuple(self.sign.shape)

    def values(self, dtype=torch.float64) -> torch.Tensor:
        return dequantize(self, dtype)


def dequantize(q: ShiftWeights, dtype=torch.float64) -> torch.Tensor:
    """sign * 2**exponent, exact (src/quant.py:142-144)."""
    return torch.ldexp(q.sign.to(dtype), q.exponent.to(torch.int32).to(dtype))


def quantize_pow2(w: torch.Tensor) -> ShiftWeights:
    """Nearest power of two, exponent clamped to [-16, 15]; zeros -> sign 0
    (src/quant.py:111-139).  Runs the CUDA quantizer."""
    w = torch.as_tensor(w)
    L.require_cuda(w)
    w = w.to(torch.float64).contiguous()
    if not bool(torch.isfinite(w).all()):
        raise ValueError("weights must be finite")
    sign = torch.empty(w.shape, dtype=torch.int8, device=w.device)
    expo = torch.empty(w.shape, dtype=torch.int8, device=w.device)
    L.run(w, "psn_quantize_pow2", L.ptr(w), w.numel(), L.ptr(sign), L.ptr(expo), L.stream_of(w))
    return ShiftWeights(sign, expo)


def _weights(w, C: int) -> torch.Tensor:
    if isinstance(w, ShiftWeights):
        w = dequantize(w)
    w = torch.as_tensor(w)
    if w.dim() != 2:
        raise ValueError(f"weights must be 2-D (channels x order), got shape {tuple(w.shape)}")
    if w.shape[0] not in (1, C):
        raise ValueError(f"weight rows {w.shape[0]} do not match {C} channels")
    return w.to(torch.float64).contiguous()


def _bias(bias, C: int, device):
    if bias is None:
        return None
    b = torch.as_tensor(bias, device=device).to(torch.float64).contiguous()
    if tuple(b.shape) != (C,):
        raise ValueError(f"bias must have shape ({C},)")
    return b


def _carrier(x: torch.Tensor) -> torch.Tensor:
    L.require_cuda(x)
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)  # reference _finish_float: non-float carriers compute as f64
    return x.contiguous()


def conv_forward(x: torch.Tensor, w, bias=None, d: int = 1) -> torch.Tensor:
    """Causal dilated channel-wise conv (src/engines.py:117-138 / 258-325).

    ``w`` as float weights runs the DIRECT engine; ``w`` as ShiftWeights runs
    the multiplication-free shift engine (ldexp on float carriers, arithmetic
    bit shifts with int64 accumulation and int32 saturation on an int32
    carrier).  Returns a tensor of the carrier dtype."""
    if d < 1:
        raise ValueError(f"dilation must be >= 1, got {d}")
    C = x.shape[2] if x.dim() >= 3 else None
    if isinstance(w, ShiftWeights) and x.dtype == torch.int32:
        out, _ = conv_forward_shift_int(x, w, bias, d)
        return out
    x = _carrier(x)
    if isinstance(w, ShiftWeights):
        sign = w.sign.to(x.device).contiguous()
        expo = w.exponent.to(x.device).contiguous()
        if sign.dim() != 2 or sign.shape[0] not in (1, C):
            raise ValueError(f"weight rows {sign.shape[0]} do not match {C} channels")
        b = _bias(bias, C, x.device)
        desc = L.make_desc(x.shape, sign.shape[1], d, x.dtype)
        out = torch.empty_like(x)
        L.run(x, "psn_conv_forward_shift", ctypes.byref(desc), L.ptr(x), L.ptr(sign), L.ptr(expo),
                                               sign.shape[0], L.ptr(b), L.ptr(out), L.stream_of(x))
        return out
    wv = _weights(w, C).to(x.device)
    b = _bias(bias, C, x.device)
    desc = L.make_desc(x.shape, wv.shape[1], d, x.dtype)
    out = torch.empty_like(x)
    L.run(x, "psn_conv_forward", ctypes.byref(desc), L.ptr(x), L.ptr(wv), wv.shape[0], L.ptr(b),
                                     L.ptr(out), L.stream_of(x))
    return out


def conv_forward_shift(x: torch.Tensor, w: ShiftWeights, bias=None, d: int = 1) -> torch.Tensor:
    """Shift engine entry point (src/engines.py:258-271)."""
    if not isinstance(w, ShiftWeights):
        raise TypeError("shift engine requires ShiftWeights")
    return conv_forward(x, w, bias, d)


def shift_spike_forward(x: torch.Tensor, w: ShiftWeights, bias=None, d: int = 1) -> torch.Tensor:
    """The quantized model layer's forward in one pass (src/network.py:352-362):
    spikes = (carrier(conv_forward_shift(x, w, bias, d)) >= 0), 0 / 1 in the
    carrier dtype (f32 or f64), bit-identical to the two-step composition."""
    if not isinstance(w, ShiftWeights):
        raise TypeError("shift engine requires ShiftWeights")
    if d < 1:
        raise ValueError(f"dilation must be >= 1, got {d}")
    x = _carrier(x)
    C = x.shape[2]
    sign = w.sign.to(x.device).contiguous()
    expo = w.exponent.to(x.device).contiguous()
    if sign.dim() != 2 or sign.shape[0] not in (1, C):
        raise ValueError(f"weight rows {sign.shape[0]} do not match {C} channels")
    b = _bias(bias, C, x.device)
    desc = L.make_desc(x.shape, sign.shape[1], d, x.dtype)
    out = torch.empty_like(x)
    L.run(x, "psn_shift_spike_forward", ctypes.byref(desc), L.ptr(x), L.ptr(sign), L.ptr(expo), sign.shape[0],
          L.ptr(b), L.ptr(out), L.stream_of(x))
    return out


def conv_forward_shift_int(x: torch.Tensor, w: ShiftWeights, bias=None, d: int = 1):
    """int32 fixed-point shift engine; returns (out int32, saturation count)
    (src/engines.py:297-325)."""
    if not isinstance(w, ShiftWeights):
        raise TypeError("shift engine requires ShiftWeights")
    L.require_cuda(x)
    if x.dtype != torch.int32:
        raise TypeError("shift_int takes an int32 carrier")
    x = x.contiguous()
    C = x.shape[2]
    sign = w.sign.to(x.device).contiguous()
    expo = w.exponent.to(x.device).contiguous()
    if sign.dim() != 2 or sign.shape[0] not in (1, C):
        raise ValueError(f"weight rows {sign.shape[0]} do not match {C} channels")
    b = _bias(bias, C, x.device)
    desc = L.make_desc(x.shape, sign.shape[1], d, torch.int32)
    out = torch.empty_like(x)
    sat = torch.zeros(1, dtype=torch.int64, device=x.device)
    L.run(x, "psn_conv_forward_shift_int", ctypes.byref(desc), L.ptr(x), L.ptr(sign), L.ptr(expo),
                                               sign.shape[0], L.ptr(b), L.ptr(out), L.ptr(sat),
                                               L.stream_of(x))
    return out, int(sat.item())


def conv_backward_input(dh: torch.Tensor, w, d: int = 1) -> torch.Tensor:
    """Time-reversed conv (src/engines.py:350-377), bit-identical to DIRECT."""
    if d < 1:
        raise ValueError(f"dilation must be >= 1, got {d}")
    dh = _carrier(dh)
    wv = _weights(w, dh.shape[2]).to(dh.device)
    desc = L.make_desc(dh.shape, wv.shape[1], d, dh.dtype)
    out = torch.empty_like(dh)
    L.run(dh, "psn_conv_backward_input", ctypes.byref(desc), L.ptr(dh), L.ptr(wv), wv.shape[0],
                                            L.ptr(out), L.stream_of(dh))
    return out


def conv_backward_weight(x: torch.Tensor, dh: torch.Tensor, k: int, d: int = 1,
                         shared: bool = False) -> torch.Tensor:
    """grad[c, i] = sum x[t-off_i] dh[t] over non-channel axes, f64
    (src/engines.py:402-425); (1, k) when shared."""
    if tuple(x.shape) != tuple(dh.shape):
        raise ValueError("input and upstream gradient must share shape and layout")
    if d < 1:
        raise ValueError(f"dilation must be >= 1, got {d}")
    dt = torch.float64 if (x.dtype == torch.float64 or dh.dtype == torch.float64) else torch.float32
    x = _carrier(x).to(dt)
    dh = _carrier(dh).to(dt)
    desc = L.make_desc(x.shape, k, d, dt)
    grad = torch.empty((1 if shared else x.shape[2], k), dtype=torch.float64, device=x.device)
    ws = L.workspace(desc, x.device)
    L.run(x, "psn_conv_backward_weight", ctypes.byref(desc), L.ptr(x), L.ptr(dh), int(bool(shared)),
                                             L.ptr(grad), L.ptr(ws), L.stream_of(x))
    return grad


def conv_backward_bias(dh: torch.Tensor) -> torch.Tensor:
    """Per-channel sum over non-channel axes, f64 (src/engines.py:428-431)."""
    dh = _carrier(dh)
    desc = L.make_desc(dh.shape, 1, 1, dh.dtype)
    grad = torch.empty(dh.shape[2], dtype=torch.float64, device=dh.device)
    ws = L.workspace(desc, dh.device)
    L.run(dh, "psn_conv_backward_bias", ctypes.byref(desc), L.ptr(dh), L.ptr(grad), L.ptr(ws),
                                           L.stream_of(dh))
    return grad

"""Neuron configuration and initialisation, mirroring the reference's
``shiftsnn.neuron`` / ``shiftsnn.quant`` / ``shiftsnn.surrogate`` config
surface for the hot path (same names, fields, defaults and errors).

Reference: src/neuron.py:21-45, 117-157; src/quant.py:18-19, 49-51;
src/surrogate.py:17-29.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

BN_EPS_DEFAULT = 1e-5
BN_MOMENTUM_DEFAULT = 0.1
E_MIN = -16
E_MAX = 15


class WeightSharing(Enum):
    CHANNEL_WISE = "channel_wise"
    SHARED = "shared"


class QuantGradMode(Enum):
    WHOLE_STE = "whole_ste"
    ROUND_STE = "round_ste"


class SurrogateKind(Enum):
    ARCTAN = "arctan"
    RATIONAL = "rational"


@dataclass(frozen=True)
class SurrogateConfig:
    kind: SurrogateKind = SurrogateKind.ARCTAN
    alpha: float = 2.0

    def __post_init__(self):
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")


@dataclass
class NeuronConfig:
    channels: int
    order: int = 2
    dilation: int = 1
    weight_sharing: WeightSharing = WeightSharing.CHANNEL_WISE
    quantized: bool = False
    grad_mode: QuantGradMode = QuantGradMode.WHOLE_STE

    def __post_init__(self):
        if self.channels < 1 or self.order < 1 or self.dilation < 1:
            raise ValueError("channels, order and dilation must all be >= 1")

    @property
    def weight_rows(self) -> int:
        return 1 if self.weight_sharing is WeightSharing.SHARED else self.channels


def sawtooth_schedule(num_layers: int) -> list[int]:
    """Dilations across a stack: 1, 2, 3, 1, 2, 3, ... (src/neuron.py:117-124)."""
    if num_layers < 1:
        raise ValueError("num_layers must be >= 1")
    out = [1]
    for _ in range(num_layers - 1):
        out.append(out[-1] % 3 + 1)
    return out


def receptive_field(orders: list[int], dilations: list[int]) -> int:
    """1 + sum (k_l - 1) d_l (src/neuron.py:127-131)."""
    if len(orders) != len(dilations):
        raise ValueError("orders and dilations must have equal length")
    return 1 + sum((k - 1) * d for k, d in zip(orders, dilations))


def tap_offsets(order: int, dilation: int) -> list[int]:
    """Offset (k-1-i)*d of tap i; tap 0 is the oldest (src/engines.py:127-130)."""
    return [(order - 1 - i) * dilation for i in range(order)]


def lif_taps(k: int, tau_m: float = 2.0) -> np.ndarray:
    """(1/tau)(1-1/tau)^(k-1-i) (src/neuron.py:134-143)."""
    if tau_m <= 1:
        raise ValueError("tau_m must be > 1")
    inv = 1.0 / tau_m
    return inv * (1.0 - inv) ** np.arange(k - 1, -1, -1, dtype=np.float64)


def init_weights(cfg: NeuronConfig, kind: str = "lif", tau_m: float = 2.0,
                 rng: np.random.Generator | None = None) -> np.ndarray:
    """Initial W of shape (rows, k), float64 (src/neuron.py:146-157).

    Uses a numpy Generator exactly like the reference, so a seeded layer here
    starts from the same weights as a seeded reference layer."""
    rows = cfg.weight_rows
    if kind == "lif":
        return np.tile(lif_taps(cfg.order, tau_m), (rows, 1))
    if kind == "uniform":
        rng = rng or np.random.default_rng()
        bound = cfg.order ** -0.5
        return rng.uniform(-bound, bound, size=(rows, cfg.order))
    raise ValueError(f"unknown init kind {kind!r}")

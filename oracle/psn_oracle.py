"""CPU oracle for the mul-free channel-wise PSN hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference ``shiftsnn`` algorithm for
exactly the path BASELINE.json's ``north_star`` names (``SpikingLayer`` TRAIN
forward + backward, plus the EVAL/shift path next to it).  It exists so the
CUDA product can be checked on the GPU box, where ``/root/reference`` does not
exist.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker or the timed CPU baseline.  Nothing in ``paper_2501_14490_b200/``
imports it; the product fails loudly when its CUDA library is missing.

Parity is PINNED: ``tests/test_oracle_golden.py`` checks every function here
bit-for-bit against vectors produced by running the reference itself
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src/shiftsnn``
in the build container and writes ``tests/golden/*.npz``), plus the
reference's own known-answer tests.

Arithmetic contract (identical to the reference, which the fixtures prove):

* convolutions accumulate in float64, tap by tap from the oldest tap
  (i = 0, offset (k-1)·d) to the newest (i = k-1, offset 0), each tap a
  separate multiply then add (no fused multiply-add), then the bias;
  result cast to the carrier dtype (f32 stays f32, f64 stays f64).
* batch statistics reduce every non-channel axis in float64 with numpy's
  two-pass mean / biased variance.
* all per-channel algebra (BN fold, running stats, gradients) is float64.

Layout: time-first ``[T, N, C, *spatial]`` (reference src/tensor.py:71-81).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# reference src/quant.py:18-22
E_MIN = -16
E_MAX = 15
INT32_MIN = -(1 << 31)
INT32_MAX = (1 << 31) - 1

# reference src/neuron.py:21-22
BN_EPS = 1e-5
BN_MOMENTUM = 0.1

# smallest double that is >= sqrt(1/2): a frexp mantissa at or above it rounds
# log2 up (sqrt(1/2) itself is irrational, so no double equals it)
_SQRT_HALF_UP = np.frombuffer(np.array([0x3FE6A09E667F3BCD], dtype=np.uint64).tobytes(),
                              dtype=np.float64)[0]


# --------------------------------------------------------------------------
# layout helpers (reference src/tensor.py:71-99)
# --------------------------------------------------------------------------

CHANNEL_AXIS = 2


def _cshape(ndim: int, n: int) -> tuple:
    s = [1] * ndim
    s[CHANNEL_AXIS] = n
    return tuple(s)


def _reduce_axes(ndim: int) -> tuple:
    return tuple(a for a in range(ndim) if a != CHANNEL_AXIS)


def _carrier(x: np.ndarray):
    """Output dtype rule of reference src/engines.py:104-106."""
    return x.dtype if x.dtype in (np.float32, np.float64) else np.float64


def tap_offsets(k: int, d: int) -> list[int]:
    """Offset of tap i is (k-1-i)*d; tap 0 is the oldest (src/engines.py:127-130)."""
    return [(k - 1 - i) * d for i in range(k)]


def sawtooth_schedule(num_layers: int) -> list[int]:
    """1,2,3,1,2,3,... (reference src/neuron.py:117-124)."""
    if num_layers < 1:
        raise ValueError("num_layers must be >= 1")
    out = [1]
    for _ in range(num_layers - 1):
        out.append(out[-1] % 3 + 1)
    return out


def receptive_field(orders, dilations) -> int:
    """1 + sum (k_l - 1) d_l (reference src/neuron.py:127-131)."""
    if len(orders) != len(dilations):
        raise ValueError("orders and dilations must have equal length")
    return 1 + sum((k - 1) * d for k, d in zip(orders, dilations))


def lif_taps(k: int, tau_m: float = 2.0) -> np.ndarray:
    """Truncated leaky-integrator kernel (reference src/neuron.py:134-143)."""
    if tau_m <= 1:
        raise ValueError("tau_m must be > 1")
    inv = 1.0 / tau_m
    return inv * (1.0 - inv) ** np.arange(k - 1, -1, -1, dtype=np.float64)


# --------------------------------------------------------------------------
# engines (reference src/engines.py)
# --------------------------------------------------------------------------

def conv_forward(x: np.ndarray, w: np.ndarray, bias=None, d: int = 1) -> np.ndarray:
    """Causal dilated channel-wise conv, DIRECT engine order.

    Follows src/engines.py:117-138 (accumulate, :132) and :109-114 (bias):
    acc = 0; for tap i oldest..newest: acc[off:] += w_i * x[:T-off]; acc += b.
    ``w`` is (C, k) or (1, k) (shared, broadcast; src/engines.py:76-92).
    """
    w = np.asarray(w, dtype=np.float64)
    if d < 1:
        raise ValueError(f"dilation must be >= 1, got {d}")
    C = x.shape[CHANNEL_AXIS]
    if w.ndim != 2 or w.shape[0] not in (1, C):
        raise ValueError(f"weight rows {w.shape} do not match {C} channels")
    if bias is not None and np.asarray(bias).shape != (C,):
        raise ValueError(f"bias must have shape ({C},)")
    T = x.shape[0]
    k = w.shape[1]
    acc = np.zeros(x.shape, dtype=np.float64)
    for i, off in enumerate(tap_offsets(k, d)):
        if off >= T:
            continue
        wi = w[:, i].reshape(_cshape(x.ndim, w.shape[0]))
        acc[off:T] += wi * x[0:T - off]
    if bias is not None:
        acc += np.asarray(bias, dtype=np.float64).reshape(_cshape(x.ndim, C))
    return acc.astype(_carrier(x), copy=False)


def conv_forward_shift_int(x: np.ndarray, sign: np.ndarray, exponent: np.ndarray,
                           bias=None, d: int = 1) -> tuple[np.ndarray, int]:
    """Fixed-point shift engine on an int32 carrier (src/engines.py:297-325).

    Per tap: ``x << e`` (e >= 0) or arithmetic ``x >> -e`` (floor), times the
    sign, accumulated in int64; bias cast to int64 (truncation toward zero,
    :318); clip to int32 at the end.  Returns (out int32, saturation count).
    """
    T = x.shape[0]
    k = sign.shape[1]
    cs = _cshape(x.ndim, sign.shape[0])
    acc = np.zeros(x.shape, dtype=np.int64)
    x64 = x.astype(np.int64)
    for i, off in enumerate(tap_offsets(k, d)):
        if off >= T:
            continue
        e = exponent[:, i].astype(np.int64).reshape(cs)
        s = sign[:, i].astype(np.int64).reshape(cs)
        src = x64[0:T - off]
        shifted = np.where(e >= 0, src << np.maximum(e, 0), src >> np.maximum(-e, 0))
        acc[off:T] += s * shifted
    if bias is not None:
        acc += np.asarray(bias, dtype=np.int64).reshape(cs)
    clipped = np.clip(acc, INT32_MIN, INT32_MAX)
    return clipped.astype(np.int32), int(np.count_nonzero(clipped != acc))


def conv_backward_input(dh: np.ndarray, w: np.ndarray, d: int = 1) -> np.ndarray:
    """Time-reversed conv, src/engines.py:350-377 (DIRECT branch):
    acc[:T-off] += w_i * dh[off:], taps oldest..newest; carrier dtype of dh."""
    w = np.asarray(w, dtype=np.float64)
    T = dh.shape[0]
    k = w.shape[1]
    acc = np.zeros(dh.shape, dtype=np.float64)
    for i, off in enumerate(tap_offsets(k, d)):
        if off >= T:
            continue
        wi = w[:, i].reshape(_cshape(dh.ndim, w.shape[0]))
        acc[0:T - off] += wi * dh[off:T]
    return acc.astype(_carrier(dh), copy=False)


def conv_backward_weight(x: np.ndarray, dh: np.ndarray, k: int, d: int = 1,
                         shared: bool = False) -> np.ndarray:
    """grad[c,i] = sum over non-channel axes of x[t-off_i] * dh[t]
    (src/engines.py:402-425); f64 product then numpy sum."""
    if x.shape != dh.shape:
        raise ValueError("input and upstream gradient must share shape")
    T = x.shape[0]
    axes = _reduce_axes(x.ndim)
    grad = np.zeros((x.shape[CHANNEL_AXIS], k), dtype=np.float64)
    xd = x.astype(np.float64, copy=False)
    dd = dh.astype(np.float64, copy=False)
    for i, off in enumerate(tap_offsets(k, d)):
        if off >= T:
            continue
        grad[:, i] = (xd[0:T - off] * dd[off:T]).sum(axis=axes)
    if shared:
        return grad.sum(axis=0, keepdims=True)
    return grad


def conv_backward_bias(dh: np.ndarray) -> np.ndarray:
    """Per-channel sum of dh over non-channel axes (src/engines.py:428-431)."""
    return dh.astype(np.float64, copy=False).sum(axis=_reduce_axes(dh.ndim))


# --------------------------------------------------------------------------
# neuron statistics (reference src/neuron.py:185-191)
# --------------------------------------------------------------------------

def batch_stats(h: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Per-channel mean and biased variance, numpy two-pass, f64."""
    axes = _reduce_axes(h.ndim)
    hd = h.astype(np.float64, copy=False)
    return hd.mean(axis=axes), hd.var(axis=axes)


# --------------------------------------------------------------------------
# quantizer (reference src/quant.py:83-144, 194-216)
# --------------------------------------------------------------------------

def quantize_pow2(w) -> tuple[np.ndarray, np.ndarray]:
    """sign(w) * 2**round(log2|w|), exponent clamped to [E_MIN, E_MAX].

    The reference (src/quant.py:111-139) rounds np.log2 and re-resolves
    borderline cases exactly (:83-108).  The nearest exponent of
    |w| = m * 2**q (m in [0.5, 1)) is q-1 when m < sqrt(1/2), else q; this
    restatement evaluates that rule directly on the frexp mantissa, which is
    the exact answer the reference's borderline resolution computes.  It is
    pinned against the reference on midpoint sweeps in the golden fixtures.
    Zero maps to (sign 0, exponent 0).
    """
    w = np.asarray(w, dtype=np.float64)
    if not np.all(np.isfinite(w)):
        raise ValueError("weights must be finite")
    sign = np.sign(w).astype(np.int8)
    m, q = np.frexp(np.abs(w))
    e = q.astype(np.int64) - 1 + (m >= _SQRT_HALF_UP)
    e = np.clip(e, E_MIN, E_MAX)
    e[w == 0.0] = 0
    return sign, e.astype(np.int8)


def dequantize(sign, exponent) -> np.ndarray:
    """sign * 2**exponent, exact (src/quant.py:142-144)."""
    return np.ldexp(np.asarray(sign).astype(np.float64), np.asarray(exponent).astype(np.int64))


def quantize_backward(g, w, round_ste: bool = False) -> np.ndarray:
    """WHOLE_STE: identity; ROUND_STE: g * |Q(w)|/|w|, zero weight -> 0
    (src/quant.py:194-216)."""
    g = np.asarray(g, dtype=np.float64)
    if not round_ste:
        return g
    w = np.asarray(w, dtype=np.float64)
    factor = np.zeros_like(w)
    nz = w != 0.0
    factor[nz] = np.abs(dequantize(*quantize_pow2(w)))[nz] / np.abs(w[nz])
    return g * factor


# --------------------------------------------------------------------------
# surrogate (reference src/surrogate.py:32-54)
# --------------------------------------------------------------------------

ARCTAN = "arctan"
RATIONAL = "rational"


def spike_backward(x, kind: str = ARCTAN, alpha: float = 2.0) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if kind == ARCTAN:
        return alpha / (2.0 * (1.0 + (0.5 * np.pi * alpha * x) ** 2))
    if kind == RATIONAL:
        return 1.0 / (1.0 + alpha * x * x)
    raise ValueError(f"unknown surrogate kind {kind!r}")


def spike_primitive(x, kind: str = ARCTAN, alpha: float = 2.0) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if kind == ARCTAN:
        return np.arctan(0.5 * np.pi * alpha * x) / np.pi + 0.5
    if kind == RATIONAL:
        r = np.sqrt(alpha)
        return np.arctan(r * x) / r + 0.5
    raise ValueError(f"unknown surrogate kind {kind!r}")


# --------------------------------------------------------------------------
# the spiking layer (reference src/network.py:143-318)
# --------------------------------------------------------------------------

@dataclass
class LayerParams:
    """Per-layer state mirrored from SpikingLayer (src/network.py:146-160)."""

    W: np.ndarray                      # (C, k) or (1, k) f64
    gamma: np.ndarray                  # (C,)
    beta: np.ndarray                   # (C,)
    running_mean: np.ndarray           # (C,)
    running_var: np.ndarray            # (C,)
    d: int = 1
    quantized: bool = True
    round_ste: bool = False
    fuse_from_batch_stats: bool = True
    quantize_in_smooth_mode: bool = False
    surrogate: str = ARCTAN
    alpha: float = 2.0
    eps: float = BN_EPS
    momentum: float = BN_MOMENTUM

    def copy(self) -> "LayerParams":
        out = LayerParams(**{k: v for k, v in self.__dict__.items()})
        for name in ("W", "gamma", "beta", "running_mean", "running_var"):
            setattr(out, name, np.array(getattr(self, name), dtype=np.float64, copy=True))
        return out

    @property
    def channels(self) -> int:
        return self.gamma.shape[0]

    def broadcast_w(self) -> np.ndarray:
        """src/network.py:197-201"""
        if self.W.shape[0] == 1 and self.channels > 1:
            return np.broadcast_to(self.W, (self.channels, self.W.shape[1]))
        return self.W


@dataclass
class ForwardCache:
    x: np.ndarray
    h1: np.ndarray
    mu: np.ndarray
    s: np.ndarray
    a: np.ndarray
    w_f: np.ndarray
    w_q: np.ndarray
    b_f: np.ndarray
    h2: np.ndarray
    use_batch: bool
    quantized: bool
    mu_batch: np.ndarray = field(default=None)
    var_batch: np.ndarray = field(default=None)


def forward_train(p: LayerParams, x: np.ndarray, smooth: bool = False):
    """TRAIN (smooth=False) / SMOOTH forward, src/network.py:236-268.

    Mutates p.running_mean / p.running_var in TRAIN mode exactly like the
    reference (:241-248).  Returns (out f64, cache).
    """
    running_prev = (p.running_mean.copy(), p.running_var.copy())
    h1 = conv_forward(x, p.W, d=p.d)
    mu_b, var_b = batch_stats(h1)
    if not smooth:
        m = h1.size // h1.shape[CHANNEL_AXIS]
        unbiased = var_b * (m / (m - 1)) if m > 1 else var_b
        mom = p.momentum
        p.running_mean *= 1 - mom
        p.running_mean += mom * mu_b
        p.running_var *= 1 - mom
        p.running_var += mom * unbiased
    use_batch = p.fuse_from_batch_stats
    mu, var = (mu_b, var_b) if use_batch else running_prev
    s = np.sqrt(var + p.eps)
    a = p.gamma / s
    w_f = a[:, None] * p.broadcast_w()
    b_f = p.beta - a * mu
    quantize = p.quantized and ((not smooth) or p.quantize_in_smooth_mode)
    w_q = dequantize(*quantize_pow2(w_f)) if quantize else w_f
    h2 = conv_forward(x, w_q, bias=b_f, d=p.d)
    if smooth:
        out = spike_primitive(h2, p.surrogate, p.alpha)
    else:
        out = (h2 >= 0).astype(np.float64)
    cache = ForwardCache(x=x, h1=h1, mu=mu, s=s, a=a, w_f=w_f, w_q=w_q, b_f=b_f,
                         h2=h2, use_batch=use_batch, quantized=quantize,
                         mu_batch=mu_b, var_batch=var_b)
    return out, cache


def backward(p: LayerParams, cache: ForwardCache, dy: np.ndarray):
    """src/network.py:272-318.  Returns (dx f64, dW, dgamma, dbeta) — the
    increments the reference accumulates into W.grad / gamma.grad / beta.grad."""
    x, h2 = cache.x, cache.h2
    d = p.d
    k = p.W.shape[1]
    shared = p.W.shape[0] == 1
    dh2 = dy * spike_backward(h2, p.surrogate, p.alpha)
    db_f = conv_backward_bias(dh2)
    dw_q = conv_backward_weight(x, dh2, k, d)
    dx = conv_backward_input(dh2, cache.w_q, d)
    dw_f = quantize_backward(dw_q, cache.w_f, p.round_ste) if cache.quantized else dw_q
    a, s, mu = cache.a, cache.s, cache.mu
    w_bc = p.broadcast_w()
    da = (dw_f * w_bc).sum(axis=1) - db_f * mu
    dw = a[:, None] * dw_f
    dbeta = db_f
    dgamma = da / s
    if cache.use_batch:
        ds = -da * p.gamma / (s * s)
        dvar = ds / (2.0 * s)
        dmu = -db_f * a
        h1 = cache.h1
        m = h1.size // h1.shape[CHANNEL_AXIS]
        cs = _cshape(h1.ndim, h1.shape[CHANNEL_AXIS])
        dh1 = (dmu / m).reshape(cs) + (2.0 / m) * dvar.reshape(cs) * (h1 - mu.reshape(cs))
        dx = dx + conv_backward_input(dh1, p.W, d)
        dw = dw + conv_backward_weight(x, dh1, k, d)
    dW = dw.sum(axis=0, keepdims=True) if shared else dw
    return dx, dW, dgamma, dbeta


def fused_running(p: LayerParams) -> tuple[np.ndarray, np.ndarray]:
    """Fold running stats into (W_f, b_f) (src/neuron.py:228-244,
    src/network.py:203-205)."""
    scale = p.gamma / np.sqrt(p.running_var + p.eps)
    w_f = np.array(p.broadcast_w()) * scale[:, None]
    b_f = p.beta - scale * p.running_mean
    return w_f, b_f


def forward_eval(p: LayerParams, x: np.ndarray) -> np.ndarray:
    """EVAL path, src/network.py:219-234 (quantized: shift engine with the
    f32-rounded fused bias; float: f32-rounded fused weights and bias)."""
    x32 = x.astype(np.float32, copy=False)
    w_f, b_f = fused_running(p)
    if p.quantized:
        w = dequantize(*quantize_pow2(w_f))
        b = b_f.astype(np.float32).astype(np.float64)
    else:
        w = w_f.astype(np.float32).astype(np.float64)
        b = b_f.astype(np.float32).astype(np.float64)
    h = conv_forward(x32, w, bias=b, d=p.d)
    return (h >= 0).astype(np.float32)


def init_layer(C: int, k: int, d: int = 1, *, weight_init: str = "lif",
               rng: np.random.Generator | None = None, shared: bool = False,
               **flags) -> LayerParams:
    """Fresh layer state as SpikingLayer.__init__ builds it
    (src/network.py:146-160, src/neuron.py:88-100, 146-157)."""
    rows = 1 if shared else C
    if weight_init == "lif":
        W = np.tile(lif_taps(k), (rows, 1))
    elif weight_init == "uniform":
        rng = rng or np.random.default_rng()
        bound = k ** -0.5
        W = rng.uniform(-bound, bound, size=(rows, k))
    else:
        raise ValueError(f"unknown init kind {weight_init!r}")
    return LayerParams(W=W, gamma=np.ones(C), beta=-np.ones(C),
                       running_mean=np.zeros(C), running_var=np.ones(C), d=d, **flags)


def train_step(p: LayerParams, x: np.ndarray, dy: np.ndarray):
    """One hot-path step (CS2): forward TRAIN then backward on dy."""
    out, cache = forward_train(p, x)
    dx, dW, dgamma, dbeta = backward(p, cache, dy)
    return out, cache, dx, dW, dgamma, dbeta


def threshold_tie_bound(x: np.ndarray, w_q: np.ndarray, b_f: np.ndarray, d: int) -> np.ndarray:
    """Per-element fp32 tie bound (SURVEY.md §8a parity fact 2):
    (k+1) * 2**-24 * (sum_i |w_q,i x[t-off_i]| + |b_f|).  An element with
    |h2_ref| below this bound is a documented threshold tie: its spike may
    legitimately differ between any two correct fp32-carrier implementations."""
    k = w_q.shape[1]
    mag = conv_forward(np.abs(x.astype(np.float64)), np.abs(w_q), bias=np.abs(b_f), d=d)
    return (k + 1) * math.ldexp(1.0, -24) * mag.astype(np.float64)

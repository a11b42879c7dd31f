"""ctypes binding of libpsn_b200.so (the C ABI declared in include/psn_b200.h).

The product path has no fallback: if the library is missing or a call fails,
this module raises.  Status codes map onto the exception types the reference
raises for the same conditions (ValueError / TypeError; RuntimeError for CUDA).
"""

from __future__ import annotations

import collections
import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSN_B200_LIB") or os.path.join(_HERE, "_lib", "libpsn_b200.so")  # PSN_B200_LIB: profiling builds (scripts/)

PSN_OK, PSN_ERR_INVALID, PSN_ERR_DTYPE, PSN_ERR_ORDER, PSN_ERR_CUDA, PSN_ERR_ALIGN = range(6)
PSN_F32, PSN_BF16, PSN_F64, PSN_I32 = range(4)
PSN_ARCTAN, PSN_RATIONAL = range(2)
PSN_QUANTIZED = 1
PSN_SHARED = 2
PSN_USE_BATCH_STATS = 4
PSN_SMOOTH = 8
PSN_QUANTIZE_IN_SMOOTH = 16
PSN_ROUND_STE = 32
PSN_GENERIC = 64
PSN_STREAM = 128
PSN_FOLD_HDR = 7


def fold_stride(k: int) -> int:
    """Doubles per channel of the forward's fold state (PSN_FOLD_STRIDE)."""
    return PSN_FOLD_HDR + 4 * int(k)

EXPORTED = (
    "psn_last_error", "psn_abi_version", "psn_max_order", "psn_fold_doubles",
    "psn_workspace_bytes", "psn_forward_train", "psn_backward", "psn_forward_eval",
    "psn_conv_forward", "psn_conv_forward_shift", "psn_conv_forward_shift_int",
    "psn_conv_backward_input", "psn_conv_backward_weight", "psn_conv_backward_bias",
    "psn_quantize_pow2", "psn_plan_info", "psn_readout_reduce", "psn_readout_expand", "psn_adam_step",
    "psn_shift_spike_forward",
)


class PsnDesc(ctypes.Structure):
    _fields_ = [
        ("T", ctypes.c_int64), ("N", ctypes.c_int64), ("C", ctypes.c_int64), ("Q", ctypes.c_int64),
        ("k", ctypes.c_int32), ("d", ctypes.c_int32), ("dtype", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("surrogate", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("alpha", ctypes.c_double), ("eps", ctypes.c_double), ("momentum", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_D = ctypes.POINTER(PsnDesc)
_SIGS = {
    "psn_last_error": (ctypes.c_char_p, []),
    "psn_abi_version": (ctypes.c_int, []),
    "psn_max_order": (ctypes.c_int, []),
    "psn_fold_doubles": (ctypes.c_size_t, [_D]),
    "psn_workspace_bytes": (ctypes.c_size_t, [_D]),
    "psn_forward_train": (ctypes.c_int, [_D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psn_backward": (ctypes.c_int, [_D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psn_forward_eval": (ctypes.c_int, [_D, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psn_conv_forward": (ctypes.c_int, [_D, _P, _P, ctypes.c_int64, _P, _P, _P]),
    "psn_conv_forward_shift": (ctypes.c_int, [_D, _P, _P, _P, ctypes.c_int64, _P, _P, _P]),
    "psn_shift_spike_forward": (ctypes.c_int, [_D, _P, _P, _P, ctypes.c_int64, _P, _P, _P]),
    "psn_conv_forward_shift_int": (ctypes.c_int, [_D, _P, _P, _P, ctypes.c_int64, _P, _P, _P, _P]),
    "psn_conv_backward_input": (ctypes.c_int, [_D, _P, _P, ctypes.c_int64, _P, _P]),
    "psn_conv_backward_weight": (ctypes.c_int, [_D, _P, _P, ctypes.c_int, _P, _P, _P]),
    "psn_conv_backward_bias": (ctypes.c_int, [_D, _P, _P, _P, _P]),
    "psn_quantize_pow2": (ctypes.c_int, [_P, ctypes.c_int64, _P, _P, _P]),
    "psn_plan_info": (ctypes.c_int, [_D, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    "psn_readout_reduce": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_double, _P, _P, _P]),
    "psn_readout_expand": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_double, _P, _P, _P]),
    "psn_adam_step": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, _P, _P]),
}

_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built — no CPU fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                        "(the PSN operators have no CPU fallback)")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == PSN_OK:
        return
    msg = lib().psn_last_error().decode(errors="replace")
    if rc in (PSN_ERR_INVALID, PSN_ERR_ORDER, PSN_ERR_ALIGN):
        raise ValueError(msg)
    if rc == PSN_ERR_DTYPE:
        raise TypeError(msg)
    raise RuntimeError(f"PSN CUDA error: {msg}")


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return PSN_F32
    if dt == torch.bfloat16:
        return PSN_BF16
    if dt == torch.float64:
        return PSN_F64
    if dt == torch.int32:
        return PSN_I32
    raise TypeError(f"unsupported carrier dtype {dt}")


def make_desc(shape, k: int, d: int, dtype: torch.dtype, flags: int = 0,
              surrogate: int = PSN_ARCTAN, alpha: float = 2.0, eps: float = 1e-5,
              momentum: float = 0.1) -> PsnDesc:
    """Descriptor for a time-first tensor of rank 3..5 ([T, N, C, *spatial])."""
    if not 3 <= len(shape) <= 5:
        raise ValueError(f"rank must be 3..5 (T, N, C plus up to 2 spatial axes), got {len(shape)}")
    T, N, C = (int(s) for s in shape[:3])
    Q = 1
    for s in shape[3:]:
        Q *= int(s)
    if min(T, N, C, Q) < 1:
        raise ValueError(f"all axis extents must be >= 1, got shape {tuple(shape)}")
    return PsnDesc(T=T, N=N, C=C, Q=Q, k=int(k), d=int(d), dtype=dtype_code(dtype), flags=int(flags),
                   surrogate=int(surrogate), reserved=0, alpha=float(alpha), eps=float(eps),
                   momentum=float(momentum))


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def run(t: torch.Tensor, name: str, *args) -> None:
    """Call C-ABI entry point `name` with t's device current (so the launch, the
    stream handle from stream_of(t) and the per-device plan attributes all refer
    to the device that owns the pointers) and raise on a non-OK status."""
    fn = getattr(lib(), name)
    with torch.cuda.device(t.device):
        rc = fn(*args)
    check(rc)


def stream_of(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def workspace(desc: PsnDesc, device) -> torch.Tensor:
    n = lib().psn_workspace_bytes(ctypes.byref(desc))
    return torch.empty(max(int(n), 256), dtype=torch.uint8, device=device)


_WS_CACHE: "collections.OrderedDict" = collections.OrderedDict()


def workspace_for(desc: PsnDesc, device, stream: int) -> torch.Tensor:
    """A persistent workspace per (device, stream, descriptor geometry).

    Saves an allocation per call; the kernels need no particular content (each
    launch zeroes its counters and accumulators)."""
    key = (torch.device(device).index, int(stream), desc.T, desc.N, desc.C, desc.Q, desc.k, desc.d,
           desc.dtype, desc.flags)
    ws = _WS_CACHE.get(key)
    if ws is None:
        ws = workspace(desc, device)
        _WS_CACHE[key] = ws
        while len(_WS_CACHE) > 32:
            _WS_CACHE.popitem(last=False)
    else:
        _WS_CACHE.move_to_end(key)
    return ws


def plan_info(desc: PsnDesc, backward: bool) -> dict:
    buf = (ctypes.c_int64 * 8)()
    n = lib().psn_plan_info(ctypes.byref(desc), int(backward), buf, 8)
    keys = ("streamed", "ctas", "groups", "tiles_per_group", "stages", "launches", "teams", "lag")
    return {k: int(buf[i]) for i, k in enumerate(keys[:n])}


def require_cuda(*tensors) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("PSN operators run on CUDA tensors only (no CPU fallback)")

PSN_MAX_ORDER_PY = 16  # mirrors PSN_MAX_ORDER in include/psn_b200.h

"""B200-native mul-free channel-wise Parallel Spiking Neuron (arXiv 2501.14490).

Drop-in for the reference ``shiftsnn`` hot path: ``SpikingLayer`` TRAIN
forward + surrogate-gradient backward (and EVAL / shift inference), with the
arithmetic in hand-written sm_100a CUDA kernels behind the C ABI of
``include/psn_b200.h``.  There is no CPU fallback.
"""

from .engines import (ShiftWeights, conv_backward_bias, conv_backward_input, conv_backward_weight,
                      conv_forward, conv_forward_shift, conv_forward_shift_int, dequantize,
                      quantize_pow2)
from .layer import Mode, ShiftLayer, SpikingLayer
from .modelio import ModelFormatError, load_model, load_tensor, save_model, save_tensor
from .net import SGD, Adam, LinearLayer, ReadoutLayer, SpikingNet, build_task_net, ce_loss
from .neuron import (BN_EPS_DEFAULT, BN_MOMENTUM_DEFAULT, E_MAX, E_MIN, NeuronConfig, QuantGradMode,
                     SurrogateConfig, SurrogateKind, WeightSharing, init_weights, lif_taps,
                     receptive_field, sawtooth_schedule, tap_offsets)

__all__ = [
    "SpikingLayer", "ShiftLayer", "Mode", "NeuronConfig", "SurrogateConfig", "SurrogateKind",
    "WeightSharing", "QuantGradMode", "ShiftWeights", "conv_forward", "conv_forward_shift",
    "conv_forward_shift_int", "conv_backward_input", "conv_backward_weight", "conv_backward_bias",
    "quantize_pow2", "dequantize", "init_weights", "lif_taps", "sawtooth_schedule",
    "receptive_field", "tap_offsets", "BN_EPS_DEFAULT", "BN_MOMENTUM_DEFAULT", "E_MIN", "E_MAX",
    "LinearLayer", "ReadoutLayer", "SpikingNet", "ce_loss", "SGD", "Adam", "build_task_net",
    "save_model", "load_model", "save_tensor", "load_tensor", "ModelFormatError",
]

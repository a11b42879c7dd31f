"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/psn_b200.h declares, and the host-side mirror of the
reference interface validates like the reference.  No compute calls."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "psn_b200.h")).read()
    return sorted(set(re.findall(r"PSN_API\s+[\w\s\*]+?\b(psn_\w+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_2501_14490_b200 import _lib as L
    assert sorted(L.EXPORTED) == _declared_symbols()


def test_library_loads_and_exports_every_symbol():
    from paper_2501_14490_b200 import _lib as L
    lib = L.lib()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    assert lib.psn_abi_version() == 2
    assert lib.psn_max_order() == L.PSN_MAX_ORDER_PY


def test_descriptor_layout_matches_c():
    from paper_2501_14490_b200 import _lib as L
    assert ctypes.sizeof(L.PsnDesc) == 80
    assert L.PsnDesc.alpha.offset == 56


def test_workspace_and_fold_sizes():
    from paper_2501_14490_b200 import _lib as L
    lib = L.lib()
    d = L.make_desc((1024, 64, 512), 4, 1, torch.float32, flags=L.PSN_QUANTIZED | L.PSN_USE_BATCH_STATS)
    assert lib.psn_fold_doubles(ctypes.byref(d)) == 512 * (7 + 4 * 4) == 512 * L.fold_stride(4)
    ws = lib.psn_workspace_bytes(ctypes.byref(d))
    assert 0 < ws < 64 << 20
    bad = L.make_desc((4, 2, 3), 17, 1, torch.float32)
    assert lib.psn_workspace_bytes(ctypes.byref(bad)) == 0  # order > 16 rejected


def test_status_codes_map_to_reference_exceptions():
    from paper_2501_14490_b200 import _lib as L
    lib = L.lib()
    d = L.make_desc((4, 2, 3), 2, 0, torch.float32)  # dilation 0
    rc = lib.psn_forward_train(ctypes.byref(d), 16, 16, 16, 16, 16, 16, 16, 16, 256, None)
    assert rc == L.PSN_ERR_INVALID
    with pytest.raises(ValueError):
        L.check(rc)
    assert b"dilation" in lib.psn_last_error()
    d = L.make_desc((4, 2, 3), 2, 1, torch.float32)
    d.dtype = 9
    with pytest.raises(TypeError):
        L.check(lib.psn_forward_train(ctypes.byref(d), 16, 16, 16, 16, 16, 16, 16, 16, 256, None))


def test_host_config_mirrors_reference():
    import paper_2501_14490_b200 as P
    with pytest.raises(ValueError):
        P.NeuronConfig(channels=0, order=1)
    with pytest.raises(ValueError):
        P.NeuronConfig(channels=1, order=1, dilation=0)
    with pytest.raises(ValueError):
        P.SurrogateConfig(alpha=0.0)
    assert P.sawtooth_schedule(6) == [1, 2, 3, 1, 2, 3]
    assert P.receptive_field([2, 2, 2], [1, 2, 3]) == 7
    assert P.tap_offsets(4, 3) == [9, 6, 3, 0]
    cfg = P.NeuronConfig(channels=5, order=3)
    assert P.init_weights(cfg).shape == (5, 3)
    u = P.init_weights(cfg, kind="uniform", rng=np.random.default_rng(0))
    assert np.all(np.abs(u) <= 3 ** -0.5)
    shared = P.NeuronConfig(channels=5, order=3, weight_sharing=P.WeightSharing.SHARED)
    assert P.init_weights(shared).shape == (1, 3)


def test_seeded_init_matches_reference_layer():
    """A seeded SpikingLayer starts from the same W as a seeded reference
    layer (both draw from numpy's Generator; golden fixture k4d1)."""
    import json
    import paper_2501_14490_b200 as P
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "manifest.json")))
    meta = [c for c in man["layer_cases"] if c["name"] == "k4d1"][0]
    z = np.load(os.path.join(ROOT, "tests", "golden", "layer_k4d1.npz"))
    cfg = P.NeuronConfig(channels=16, order=4, dilation=1, quantized=True)
    w = P.init_weights(cfg, kind="uniform", rng=np.random.default_rng(meta["seed"] + 1))
    assert np.array_equal(w, z["W"])


def test_product_has_no_cpu_fallback():
    import paper_2501_14490_b200 as P
    layer = P.SpikingLayer(P.NeuronConfig(channels=4, order=2), device="cpu")
    with pytest.raises(ValueError, match="CUDA"):
        layer(torch.zeros(3, 2, 4), P.Mode.TRAIN)
    with pytest.raises(ValueError, match="CUDA"):
        P.conv_forward(torch.zeros(3, 2, 4, dtype=torch.float64), torch.ones(4, 2, dtype=torch.float64))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2501_14490_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f

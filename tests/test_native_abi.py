"""CPU checks of the C-ABI boundary: the in-tree library loads without a GPU and exports
every entry point include/dart_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

from paper_2603_11441_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "dart_b200.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(dart_\w+)\s*\(", text, flags=re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libdart_b200.so not built")
    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.dart_version()


def test_weight_count_matches_declaration():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libdart_b200.so not built")
    import paper_2603_11441_b200 as D
    from paper_2603_11441_b200.model import param_declaration

    lib = _native.load()
    for cfg in (D.toy_config(), D.vit_h_config()):
        desc = _native.ModelDesc()
        desc.num_blocks = cfg.num_blocks
        desc.num_encoder_layers = cfg.num_encoder_layers
        desc.num_decoder_layers = cfg.num_decoder_layers
        assert lib.dart_expected_weight_count(ctypes.byref(desc)) == len(param_declaration(cfg, False))


def test_no_cuda_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2603_11441_b200 as D

    model = D.build_model(D.toy_config(), with_mask_head=False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        D.backbone_forward(model, np.zeros((64, 64, 3)))

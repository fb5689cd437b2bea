"""CPU-side checks of the C-ABI boundary: the library loads without a GPU,
exports exactly what include/vchitect_b200.h declares, and its pure
size/shape queries behave (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

from paper_2501_08453_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vchitect_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"VC_API\s+[\w\s\*]+?\b(vc_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"


def test_version_and_shape_queries():
    lib = _lib.load()
    assert b"sm_100a" in lib.vc_version()
    s = _lib.shape(16, 1350, 256, 1584, 24, "bf16")
    assert lib.vc_block_shape_check(C.byref(s)) == 0
    D = 1584
    assert lib.vc_block_raw_weight_floats(C.byref(s)) == 3 * (2 * D + 4 * D * D)
    assert lib.vc_block_packed_weight_bytes(C.byref(s)) >= 12 * D * D * 2
    assert lib.vc_block_workspace_bytes(C.byref(s)) > 0
    assert lib.vc_block_host_workspace_bytes(C.byref(s)) > lib.vc_block_workspace_bytes(C.byref(s))
    assert lib.vc_block_forward_launches(C.byref(s)) > 0


@pytest.mark.parametrize("args", [(2, 5, 1, 12, 5, "fp32"), (0, 5, 1, 12, 4, "fp32"),
                                  (2, 5, 1, 20, 4, "bf16")])
def test_shape_errors_are_einval(args):
    lib = _lib.load()
    s = _lib.shape(*args)
    assert lib.vc_block_shape_check(C.byref(s)) == _lib.VC_EINVAL
    with pytest.raises(ValueError):
        _lib.check(lib.vc_block_shape_check(C.byref(s)))
    assert b"" != lib.vc_last_error()


def test_divisibility_message_matches_reference_wording():
    lib = _lib.load()
    s = _lib.shape(2, 5, 1, 12, 5, "fp32")
    lib.vc_block_shape_check(C.byref(s))
    assert b"not divisible by 5 heads" in lib.vc_last_error()


def test_compute_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2501_08453_b200 import attention
    with pytest.raises(RuntimeError):
        attention(np.zeros((2, 4)), np.zeros((2, 4)), np.zeros((2, 4)), 2)

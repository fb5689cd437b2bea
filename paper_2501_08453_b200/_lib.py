"""ctypes binding of the in-tree C-ABI library (include/vchitect_b200.h).

The library is the product: there is no Python or CPU fallback. Loading
fails loudly if libvchitect_b200.so has not been built, and every compute
entry point refuses to run without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvchitect_b200.so")

VC_OK = 0
VC_EINVAL = -22
VC_ECUDA = -1000
VC_ENOTSUP = -95
DTYPES = {"fp32": 0, "bf16": 1}


class BlockShape(C.Structure):
    _fields_ = [("frames", C.c_int32), ("visual_len", C.c_int32), ("text_len", C.c_int32),
                ("dim", C.c_int32), ("heads", C.c_int32), ("dtype", C.c_int32)]


class ExtShape(C.Structure):
    _fields_ = [("block", BlockShape), ("grid_h", C.c_int32), ("grid_w", C.c_int32),
                ("ffn_dim", C.c_int32)]


class SpPlan(C.Structure):
    _fields_ = [("shape", BlockShape), ("nranks", C.c_int32), ("rank", C.c_int32)]


# name -> (restype, argtypes); mirrors include/vchitect_b200.h one to one.
_p, _f, _i32, _i64, _sz, _d = C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_size_t, C.c_double
_S = C.POINTER(BlockShape)
SIGNATURES = {
    "vc_version": (C.c_char_p, []),
    "vc_last_error": (C.c_char_p, []),
    "vc_block_shape_check": (C.c_int, [_S]),
    "vc_block_raw_weight_floats": (_sz, [_S]),
    "vc_block_packed_weight_bytes": (_sz, [_S]),
    "vc_block_workspace_bytes": (_sz, [_S]),
    "vc_pack_block_weights": (C.c_int, [_S, _p, _p, _p]),
    "vc_block_forward": (C.c_int, [_S, _p, _p, _p, _p, C.c_int, _p, _sz, _p]),
    "vc_block_host_workspace_bytes": (_sz, [_S]),
    "vc_block_forward_host": (C.c_int, [_S, _p, _p, _p, _p, _p, _sz, _p]),
    "vc_block_stream_workspace_bytes": (_sz, [_S]),
    "vc_block_forward_host_batched": (C.c_int, [_S, _p, _i32, C.POINTER(C.c_void_p), _p,
                                                C.POINTER(C.c_void_p), _p, _sz, _p, _p, _p]),
    "vc_attention_f32": (C.c_int, [_p, _p, _p, _p, _i32, _i32, _i32, _i32, _p]),
    "vc_attention_bf16_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32]),
    "vc_attention_bf16": (C.c_int, [_p, _p, _p, _p, _i32, _i32, _i32, _i32, _i32, C.c_float, _p, _sz, _p]),
    "vc_layer_norm_f32": (C.c_int, [_p, _p, _i64, _i32, _p]),
    "vc_embed_frames": (C.c_int, [_p, _p, _p, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _d, _p]),
    "vc_unembed_frames": (C.c_int, [_p, _p, _p, _i32, _i32, _i32, _i32, _i32, _i32, _p]),
    "vc_unembed_reverse_step": (C.c_int, [_p, _p, _p, _p, _p, _p, _i32, _i32, _i32, _i32, _i32, _i32,
                                          _d, _d, _d, _p]),
    "vc_embed_frames_rows": (C.c_int, [_p, _p, _p, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _d, _p]),
    "vc_gemm_bf16": (C.c_int, [_p, _i64, _p, _i64, _p, _p, _p, _i64, _i64, _i32, _i32, _p]),
    "vc_block_forward_launches": (C.c_int, [_S]),
    "vc_sp_check": (C.c_int, [C.POINTER(SpPlan)]),
    "vc_sp_bounds": (C.c_int, [C.POINTER(SpPlan), C.POINTER(C.c_int32)]),
    "vc_sp_workspace_bytes": (_sz, [C.POINTER(SpPlan)]),
    "vc_sp_exchange_elems": (_i64, [C.POINTER(SpPlan), _i32, _i32]),
    "vc_sp_row_map": (_i32, [C.POINTER(SpPlan), _i32, C.c_void_p]),
    "vc_vae_encode_frames": (_i32, [_p, _p, _p, _i32, _i32, _i32, _i32, _i32, _d, _d, _p]),
    "vc_sp_reshard_elems": (_i64, [C.POINTER(SpPlan), _i32, _i32]),
    "vc_sp_reshard_pack": (_i32, [C.POINTER(SpPlan), _p, _p, _p]),
    "vc_sp_reshard_unpack": (_i32, [C.POINTER(SpPlan), _p, _p, _p]),
    "vc_set_temporal_impl": (C.c_int, [_i32]),
    "vc_sp_stage1": (C.c_int, [C.POINTER(SpPlan), _p, _p, _p, _p, _p, _sz, _p]),
    "vc_sp_stage1_part": (C.c_int, [C.POINTER(SpPlan), _p, _p, _p, _p, _i32, _p, _sz, _p]),
    "vc_sp_stage2": (C.c_int, [C.POINTER(SpPlan), _p, _p, _p, _p, _sz, _p]),
    "vc_sp_stage2_branch": (C.c_int, [C.POINTER(SpPlan), _p, _p, _p, _i32, _p, _sz, _p]),
    "vc_sp_stage3": (C.c_int, [C.POINTER(SpPlan), _p, _p, _p, _p, C.c_int, _p, _sz, _p]),
    "vc_spg_check": (C.c_int, [C.POINTER(SpPlan)]),
    "vc_spg_workspace_bytes": (_sz, [C.POINTER(SpPlan)]),
    "vc_spg_slot_elems": (_i64, [C.POINTER(SpPlan)]),
    "vc_spg_stage1": (C.c_int, [C.POINTER(SpPlan), _p, _p, _p, _p, _p, _sz, _p]),
    "vc_spg_stage2": (C.c_int, [C.POINTER(SpPlan), _p, _p, _p, _p, C.c_int, _p, _sz, _p]),
    "vc_ext_raw_weight_floats": (_sz, [C.POINTER(ExtShape)]),
    "vc_ext_packed_weight_bytes": (_sz, [C.POINTER(ExtShape)]),
    "vc_pack_ext_weights": (C.c_int, [C.POINTER(ExtShape), _p, _p, _p]),
    "vc_ext_workspace_bytes": (_sz, [C.POINTER(ExtShape)]),
    "vc_ext_block_forward": (C.c_int, [C.POINTER(ExtShape), _p, _p, _p, _p, _d, _p, _p, _sz, _p]),
    "vc_ext_block_launches": (C.c_int, [C.POINTER(ExtShape)]),
    "vc_profile_enable": (C.c_int, [C.c_int]),
    "vc_profile_reset": (None, []),
    "vc_profile_read": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_int32, C.c_char_p, C.c_size_t]),
}

_lib = None


def load():
    """Load the library (no GPU needed to load or to query sizes)."""
    global _lib
    if _lib is None:
        # VC_LIB_PATH: A/B aid for profiling two builds on one box (tools/)
        path = os.environ.get("VC_LIB_PATH", LIB_PATH)
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -m paper_2501_08453_b200.build` "
                "(the CUDA path has no fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == VC_OK:
        return
    msg = load().vc_last_error().decode(errors="replace")
    if rc == VC_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"{what or 'vchitect_b200'} failed ({rc}): {msg}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_08453_b200 needs a CUDA B200 (sm_100a); there is no CPU path")
    return torch


def shape(frames, visual_len, text_len, dim, heads, dtype="fp32") -> BlockShape:
    if dtype not in DTYPES:
        raise ValueError(f"dtype must be one of {tuple(DTYPES)}, got {dtype!r}")
    return BlockShape(int(frames), int(visual_len), int(text_len), int(dim), int(heads), DTYPES[dtype])


def stream_ptr(torch, stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)

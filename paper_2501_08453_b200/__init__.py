"""B200-native parallel MM-DiT block forward (Vchitect-2.0, arXiv 2501.08453).

Drop-in for the reference `spsim` hot path: `parallel_block_forward`,
the branch functions, `ToyDenoiser` and `attention`, computed by
hand-written sm_100a CUDA kernels behind the C ABI in
include/vchitect_b200.h (libvchitect_b200.so, loaded with ctypes).
"""
from .model import (  # noqa: F401
    BlockParams,
    BranchParams,
    PatchSpec,
    ToyDenoiser,
    anchor_text,
    branch_attention,
    full_sequence_attention,
    layer_norm,
    parallel_block_forward,
    seq_len,
    spatial_branch,
    temporal_branch,
    toy_vae_encode,
)
from .numerics import SeededRng, attention  # noqa: F401

__all__ = [
    "BlockParams", "BranchParams", "PatchSpec", "ToyDenoiser", "SeededRng", "anchor_text",
    "attention", "branch_attention", "full_sequence_attention", "layer_norm",
    "parallel_block_forward", "seq_len", "spatial_branch", "temporal_branch",
]

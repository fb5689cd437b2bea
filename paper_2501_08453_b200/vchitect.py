"""The north-star extensions of the block: AdaLN timestep modulation,
QK-RMSNorm + 3D RoPE fused into the Q/K projection epilogue, and the gated
GELU FFN (BASELINE.json north_star; SURVEY.md §8 "a-ext").

The reference `spsim` block (model.py:263-271) has none of these, so there is
nothing to be a drop-in for and the parity is UNPINNED: the semantics are the
ones oracle/vchitect_ext_oracle.py states, and tests/test_gpu_ext.py checks
this path against that oracle. The block API follows north_star's
`forward(x_video, text_emb, timestep)`; the reference-semantics API
(`parallel_block_forward`, `ToyDenoiser`, ...) is untouched by it.

    params = VchitectExtParams.init(SeededRng(0), dim=1584, heads=24)
    blk = VchitectBlock(params, heads=24, grid=(30, 45))
    y = blk.forward(x_video, text_emb, timestep)   # [F, Lv, D], residuals included

Runs on the bf16 tensor-core path only (vc_ext_block_forward).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .model import BlockParams, DeviceBlock, workspace
from .numerics import SeededRng, _is_torch, to_device_f32


@dataclass
class VchitectExtParams:
    """The reference BlockParams plus the extension weights. Draw order from
    rng.split(404): w_ada, b_ada, q_norm[2, dh], k_norm[2, dh] (rows: spatial,
    full sequence), w1, b1, w2, b2; the block from rng.split(1000)."""
    block: BlockParams
    w_ada: np.ndarray   # [D, 6D]
    b_ada: np.ndarray   # [6D]
    q_norm: np.ndarray  # [2, dh]
    k_norm: np.ndarray  # [2, dh]
    w1: np.ndarray      # [D, Dff]
    b1: np.ndarray      # [Dff]
    w2: np.ndarray      # [Dff, D]
    b2: np.ndarray      # [D]

    @staticmethod
    def init(rng: SeededRng, dim: int, heads: int, mlp_ratio: float = 2.0) -> "VchitectExtParams":
        if dim % heads:
            raise ValueError(f"feature dim {dim} not divisible by {heads} heads")
        dh = dim // heads
        dff = int(round(dim * mlp_ratio))
        block = BlockParams.init(rng.split(1000), dim)
        e = rng.split(404)
        w_ada = 0.5 / math.sqrt(dim) * e.normal((dim, 6 * dim))
        b_ada = 0.02 * e.normal(6 * dim)
        q_norm = 1.0 + 0.02 * e.normal((2, dh))
        k_norm = 1.0 + 0.02 * e.normal((2, dh))
        w1 = e.normal((dim, dff)) / math.sqrt(dim)
        b1 = 0.02 * e.normal(dff)
        w2 = e.normal((dff, dim)) / math.sqrt(dff)
        b2 = 0.02 * e.normal(dim)
        return VchitectExtParams(block, w_ada, b_ada, q_norm, k_norm, w1, b1, w2, b2)

    def ext_arrays(self):
        return (self.w_ada, self.b_ada, self.q_norm, self.k_norm, self.w1, self.b1, self.w2, self.b2)


def ext_shape(frames, visual_len, text_len, dim, heads, grid, ffn_dim) -> _lib.ExtShape:
    gh, gw = grid
    return _lib.ExtShape(_lib.shape(frames, visual_len, text_len, dim, heads, "bf16"),
                         int(gh), int(gw), int(ffn_dim))


class VchitectBlock:
    """Device handle: packed block + extension weights, the forward call."""

    def __init__(self, params: VchitectExtParams, heads: int, grid):
        torch = _lib.require_cuda()
        dim = params.block.spatial.wq.shape[0]
        self.heads, self.dim, self.grid = heads, dim, (int(grid[0]), int(grid[1]))
        self.ffn_dim = params.w1.shape[1]
        if params.w1.shape != (dim, self.ffn_dim) or params.w2.shape != (self.ffn_dim, dim):
            raise ValueError("FFN weights do not match the block dim")
        self.db = DeviceBlock(torch, params.block, heads, "bf16")
        lib = _lib.load()
        shp = ext_shape(1, self.grid[0] * self.grid[1], 0, dim, heads, self.grid, self.ffn_dim)
        n = lib.vc_ext_raw_weight_floats(C.byref(shp))
        if n == 0:
            raise ValueError((lib.vc_last_error() or b"").decode())
        raw = np.concatenate([np.ascontiguousarray(a, dtype=np.float32).ravel() for a in params.ext_arrays()])
        if raw.size != n:
            raise ValueError(f"extension weights hold {raw.size} floats, expected {n}")
        self.packed = torch.empty(lib.vc_ext_packed_weight_bytes(C.byref(shp)), dtype=torch.uint8, device="cuda")
        raw_t = torch.from_numpy(raw).cuda()
        _lib.check(lib.vc_pack_ext_weights(C.byref(shp), _lib.ptr(raw_t), _lib.ptr(self.packed),
                                           _lib.stream_ptr(torch)), "pack extension weights")
        torch.cuda.current_stream().synchronize()

    def shape(self, frames, visual_len, text_len):
        return ext_shape(frames, visual_len, text_len, self.dim, self.heads, self.grid, self.ffn_dim)

    def forward_device(self, x, prompt, timestep, out, stream=None):
        """x/out [F, Lv, D] fp32 CUDA (distinct), prompt [Lt, D] fp32 CUDA or None."""
        torch = _lib.require_cuda()
        F, Lv, D = x.shape
        Lt = prompt.shape[0] if prompt is not None else 0
        lib = _lib.load()
        shp = self.shape(F, Lv, Lt)
        nbytes = lib.vc_ext_workspace_bytes(C.byref(shp))
        if nbytes == 0:
            raise ValueError((lib.vc_last_error() or b"").decode())
        ws = workspace(torch, nbytes)
        _lib.check(lib.vc_ext_block_forward(C.byref(shp), _lib.ptr(self.db.packed), _lib.ptr(self.packed),
                                            _lib.ptr(x), _lib.ptr(prompt) if Lt else C.c_void_p(0),
                                            float(timestep), _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                            _lib.stream_ptr(torch, stream)), "extended block forward")
        return out

    def forward(self, x_video, text_emb, timestep):
        """north_star's forward(x_video, text_emb, timestep): x_video
        [F, Lv, D]; text_emb [F, Lt, D] (anchored: frame 0's text is used for
        every frame, model.py:257) or [Lt, D]; returns [F, Lv, D] (numpy in,
        numpy out; CUDA tensors in, CUDA tensor out)."""
        torch = _lib.require_cuda()
        if x_video.ndim != 3 or x_video.shape[2] != self.dim:
            raise ValueError(f"x_video must be [frames, len, {self.dim}]")
        if x_video.shape[1] != self.grid[0] * self.grid[1]:
            raise ValueError(f"grid {self.grid} does not hold {x_video.shape[1]} tokens")
        prompt = text_emb[0] if text_emb.ndim == 3 else text_emb
        if prompt.ndim != 2 or (prompt.shape[0] and prompt.shape[1] != self.dim):
            raise ValueError("text_emb must be [frames, len, dim] or [len, dim]")
        as_numpy = not _is_torch(x_video)
        x = to_device_f32(torch, x_video)
        p = to_device_f32(torch, prompt) if prompt.shape[0] else None
        out = torch.empty_like(x)
        self.forward_device(x, p, timestep, out)
        return out.double().cpu().numpy() if as_numpy else out

    __call__ = forward

"""Drop-in for spsim.numerics on the hot path (numerics.py in the reference).

`SeededRng` is the host-side weight / input generator (same Philox stream
and XOR-split derivation as numerics.py:38-69, so "same random-init
weights" holds bit for bit). `attention` runs the fp32 SIMT kernel through
the C ABI (vc_attention_f32); it accepts numpy (returns numpy float64) or
CUDA torch tensors (returns a CUDA float32 tensor).
"""
from __future__ import annotations

import numpy as np

from . import _lib

_MASK64 = (1 << 64) - 1
RNG_ALGORITHM = "philox4x64-v1"


class SeededRng:
    """Counter-based stream; substreams by seed XOR tag (numerics.py:38-69)."""

    algorithm = RNG_ALGORITHM

    def __init__(self, seed: int):
        self.seed = int(seed) & _MASK64
        self._gen = np.random.Generator(np.random.Philox(key=self.seed))

    def split(self, tag: int) -> "SeededRng":
        return SeededRng(self.seed ^ (int(tag) & _MASK64))

    def normal(self, shape=()):
        return self._gen.standard_normal(size=shape, dtype=np.float64)

    def uniform(self, shape=()):
        return self._gen.random(size=shape, dtype=np.float64)

    def integers(self, low, high, shape=()):
        return self._gen.integers(low, high, size=shape)


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def to_device_f32(torch, a):
    """numpy / torch -> contiguous CUDA float32 tensor."""
    if _is_torch(a):
        t = a
        if not t.is_cuda:
            t = t.cuda()
        return t.to(torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def attention(q, k, v, heads: int, *, dtype: str = "fp32", weighted_keys=None):
    """Multi-head SDPA on [s, d] inputs (numerics.py:87-107), on the GPU.

    dtype "fp32": FFMA SIMT kernel (1e-4 class); "bf16": the tcgen05 tensor-core
    kernel the block runs (2e-2 class, head dims up to 128).  weighted_keys =
    (n, w) gives the first n keys multiplicity w (logit + log w) -- the
    deduplicated anchored text of the full-sequence branch (bf16 only)."""
    torch = _lib.require_cuda()
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise ValueError("attention expects 2-D q/k/v")
    s, d = q.shape
    if tuple(k.shape) != tuple(v.shape) or k.shape[1] != d:
        raise ValueError(f"q/k/v shapes disagree: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    if d % heads != 0:
        raise ValueError(f"feature dim {d} not divisible by {heads} heads")
    if dtype not in ("fp32", "bf16"):
        raise ValueError(f"dtype must be 'fp32' or 'bf16', got {dtype!r}")
    if weighted_keys is not None and dtype != "bf16":
        raise ValueError("weighted_keys needs dtype='bf16'")
    as_numpy = not _is_torch(q)
    tq, tk, tv = (to_device_f32(torch, a) for a in (q, k, v))
    out = torch.empty_like(tq)
    lib = _lib.load()
    if dtype == "fp32":
        _lib.check(lib.vc_attention_f32(_lib.ptr(tq), _lib.ptr(tk), _lib.ptr(tv), _lib.ptr(out),
                                        s, k.shape[0], d, heads, _lib.stream_ptr(torch)), "attention")
    else:
        n_w, w = weighted_keys if weighted_keys is not None else (0, 1.0)
        nbytes = int(lib.vc_attention_bf16_workspace_bytes(s, k.shape[0], d, heads))
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        _lib.check(lib.vc_attention_bf16(_lib.ptr(tq), _lib.ptr(tk), _lib.ptr(tv), _lib.ptr(out), s, k.shape[0], d,
                                         heads, int(n_w), float(w), _lib.ptr(ws), nbytes, _lib.stream_ptr(torch)),
                   "attention")
    if as_numpy:
        return out.double().cpu().numpy()
    return out

"""Drop-in for the reference block / model API (spsim.model), on B200.

Same names, argument order, weight layout and ValueError behaviour as
/root/reference/pkg/src/spsim/model.py; the compute runs in the C-ABI
library (include/vchitect_b200.h) on the GPU:

  parallel_block_forward(block, visual, text, heads)    model.py:263-271
  spatial_branch / temporal_branch / full_sequence_attention / branch_attention
                                                         model.py:187-260
  ToyDenoiser.init / embed_frame / head_states / forward model.py:274-333
  BranchParams.init / BlockParams.init                   model.py:157-205

Inputs may be numpy (returns numpy float64, the reference's value semantics)
or CUDA torch tensors (returns CUDA float32 tensors, no host round trip).
Every compute function takes a keyword-only `dtype` ("fp32" -- FFMA, the
1e-4 parity path -- or "bf16" -- tcgen05 tensor cores, the 2e-2 path);
the default is module-level DEFAULT_DTYPE.

Params stay host numpy arrays (mutable, as in the reference: its tests
mutate model.w_out in place). Device copies are cached per object and
re-packed when a content fingerprint (xor of the float64 bit patterns)
changes, so in-place mutation is always seen.
"""
from __future__ import annotations

import ctypes as C
import weakref
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .numerics import SeededRng, _is_torch, to_device_f32

DEFAULT_DTYPE = "fp32"


# ---------------------------------------------------------------------------
# Geometry and host-side helpers (pure index maps; model.py:28-154)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class PatchSpec:
    """model.py:28-43."""
    vae_downsample: int = 8
    patch: int = 2
    latent_channels: int = 4

    def latent_hw(self, height: int, width: int):
        d = self.vae_downsample
        return (math.ceil(height / d), math.ceil(width / d))

    def tokens_per_frame(self, height: int, width: int) -> int:
        h, w = self.latent_hw(height, width)
        return math.ceil(h / self.patch) * math.ceil(w / self.patch)


def seq_len(frames: int, height: int, width: int, spec: PatchSpec = PatchSpec()) -> int:
    """model.py:46-50."""
    if frames < 1 or height < 1 or width < 1:
        raise ValueError(f"bad clip shape ({frames}, {height}, {width})")
    return frames * spec.tokens_per_frame(height, width)


def anchor_text(prompt, frames: int):
    """model.py:126-130: broadcast one prompt into every frame's text slots."""
    if prompt.ndim != 2:
        raise ValueError("prompt must be [len, dim]")
    if _is_torch(prompt):
        return prompt.unsqueeze(0).expand(frames, *prompt.shape).contiguous()
    return np.broadcast_to(prompt, (frames,) + prompt.shape).copy()


# ---------------------------------------------------------------------------
# Parameters (host numpy, reference layout and init streams)
# ---------------------------------------------------------------------------

@dataclass
class BranchParams:
    """model.py:157-178 -- gamma, beta [D]; wq, wk, wv, wo [D_in, D_out]."""
    gamma: np.ndarray
    beta: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray

    @staticmethod
    def init(rng: SeededRng, dim: int) -> "BranchParams":
        s = 1.0 / math.sqrt(dim)
        gamma = 1.0 + 0.02 * rng.normal(dim)
        beta = 0.02 * rng.normal(dim)
        wq = s * rng.normal((dim, dim))
        wk = s * rng.normal((dim, dim))
        wv = s * rng.normal((dim, dim))
        wo = s * rng.normal((dim, dim))
        return BranchParams(gamma, beta, wq, wk, wv, wo)

    @staticmethod
    def zeros(dim: int) -> "BranchParams":
        """A branch whose output is exactly zero (W = 0)."""
        z = np.zeros((dim, dim))
        return BranchParams(np.ones(dim), np.zeros(dim), z, z, z, z)

    def arrays(self):
        return (self.gamma, self.beta, self.wq, self.wk, self.wv, self.wo)


@dataclass
class BlockParams:
    """model.py:193-205 -- branch streams split(101/202/303)."""
    spatial: BranchParams
    temporal: BranchParams
    fullseq: BranchParams

    @staticmethod
    def init(rng: SeededRng, dim: int) -> "BlockParams":
        return BlockParams(
            spatial=BranchParams.init(rng.split(101), dim),
            temporal=BranchParams.init(rng.split(202), dim),
            fullseq=BranchParams.init(rng.split(303), dim),
        )

    def branches(self):
        return (self.spatial, self.temporal, self.fullseq)


def _fingerprint(arrays):
    fp = []
    for a in arrays:
        a64 = np.ascontiguousarray(a, dtype=np.float64)
        fp.append((a.shape, int(np.bitwise_xor.reduce(a64.view(np.uint64).ravel())) if a64.size else 0))
    return tuple(fp)


class DeviceBlock:
    """Packed device weights of one BlockParams (vc_pack_block_weights)."""

    def __init__(self, torch, block: BlockParams, heads: int, dtype: str):
        dim = block.spatial.wq.shape[0]
        raw = np.concatenate([np.ascontiguousarray(a, dtype=np.float32).ravel()
                              for br in block.branches() for a in br.arrays()])
        lib = _lib.load()
        self.shape = _lib.shape(1, 1, 0, dim, heads, dtype)
        _lib.check(lib.vc_block_shape_check(C.byref(self.shape)), "block shape")
        if raw.size != lib.vc_block_raw_weight_floats(C.byref(self.shape)):
            raise ValueError(f"block weights do not match dim {dim}")
        nbytes = lib.vc_block_packed_weight_bytes(C.byref(self.shape))
        self.packed = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        raw_t = torch.from_numpy(raw).cuda()
        _lib.check(lib.vc_pack_block_weights(C.byref(self.shape), _lib.ptr(raw_t),
                                             _lib.ptr(self.packed), _lib.stream_ptr(torch)), "pack")
        self.dim, self.heads, self.dtype = dim, heads, dtype
        self.fingerprint = _fingerprint([a for br in block.branches() for a in br.arrays()])


_BLOCK_CACHE: dict = {}
_WS = {"buf": None}


def device_block(torch, block: BlockParams, heads: int, dtype: str) -> DeviceBlock:
    key = (id(block), heads, dtype)
    fp = _fingerprint([a for br in block.branches() for a in br.arrays()])
    hit = _BLOCK_CACHE.get(key)
    if hit is not None and hit[0]() is block and hit[1].fingerprint == fp:
        return hit[1]
    db = DeviceBlock(torch, block, heads, dtype)
    # weak reference: the cache must not keep a BlockParams (and its device
    # weights) alive; the entry is dropped when the block is collected
    _BLOCK_CACHE[key] = (weakref.ref(block), db)
    weakref.finalize(block, _BLOCK_CACHE.pop, key, None)
    return db


def workspace(torch, nbytes: int):
    buf = _WS["buf"]
    if buf is None or buf.numel() < nbytes:
        _WS["buf"] = None
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        _WS["buf"] = buf
    return buf


def _resolve_dtype(dtype):
    d = DEFAULT_DTYPE if dtype is None else dtype
    if d not in _lib.DTYPES:
        raise ValueError(f"dtype must be one of {tuple(_lib.DTYPES)}, got {d!r}")
    return d


def block_forward_device(torch, db: DeviceBlock, x, prompt, out, add_residual: bool, stream=None):
    """Raw device call: x/out [F, Lv, D] fp32 CUDA, prompt [Lt, D] fp32 CUDA."""
    F, Lv, D = x.shape
    Lt = prompt.shape[0] if prompt is not None else 0
    lib = _lib.load()
    shp = _lib.shape(F, Lv, Lt, D, db.heads, db.dtype)
    nbytes = lib.vc_block_workspace_bytes(C.byref(shp))
    if nbytes == 0:
        _lib.check(lib.vc_block_shape_check(C.byref(shp)), "shape")
    ws = workspace(torch, nbytes)
    _lib.check(lib.vc_block_forward(C.byref(shp), _lib.ptr(db.packed), _lib.ptr(x),
                                    _lib.ptr(prompt) if Lt else C.c_void_p(0), _lib.ptr(out),
                                    1 if add_residual else 0, _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr(torch, stream)), "block forward")
    return out


# ---------------------------------------------------------------------------
# Block and branch forwards
# ---------------------------------------------------------------------------

def _check_visual(visual, text=None):
    if visual.ndim != 3:
        raise ValueError("visual must be [frames, len, dim]")
    if text is not None:
        if text.ndim != 3:
            raise ValueError("text must be [frames, len, dim]")
        if text.shape[2] != visual.shape[2]:
            raise ValueError("text and visual feature dims disagree")


def parallel_block_forward(block: BlockParams, visual, text, heads: int, *, dtype=None):
    """Sum of the three branches (model.py:263-271). The caller adds the residual."""
    _check_visual(visual, text)
    torch = _lib.require_cuda()
    dtype = _resolve_dtype(dtype)
    D = visual.shape[2]
    if D % heads != 0:
        raise ValueError(f"feature dim {D} not divisible by {heads} heads")
    as_numpy = not _is_torch(visual)
    x = to_device_f32(torch, visual)
    prompt = to_device_f32(torch, text[0]) if text.shape[1] > 0 else None
    db = device_block(torch, block, heads, dtype)
    out = torch.empty_like(x)
    block_forward_device(torch, db, x, prompt, out, False)
    return out.double().cpu().numpy() if as_numpy else out


def block_forward_host_stream(block, visuals, prompt, heads: int, outs=None, *, dtype=None):
    """Serving path: parallel_block_forward over a list of HOST batches (pinned
    float32 torch tensors [F, Lv, D]) with one shared prompt [Lt, D], through
    vc_block_forward_host_batched: H2D of batch i+1 and D2H of batch i-1
    overlap the compute of batch i. Returns the list of host outputs.

    `block` is a BlockParams (packed to the device on first use and re-packed
    when its arrays change) or a DeviceBlock — the device-resident weight
    handle a server keeps, which skips the per-call host-side change check."""
    torch = _lib.require_cuda()
    if isinstance(block, DeviceBlock):
        db = block
        if heads != db.heads or (dtype is not None and _resolve_dtype(dtype) != db.dtype):
            raise ValueError("heads / dtype disagree with the DeviceBlock")
        dtype = db.dtype
    else:
        dtype = _resolve_dtype(dtype)
        db = device_block(torch, block, heads, dtype)
    F, Lv, D = visuals[0].shape
    Lt = prompt.shape[0]
    lib = _lib.load()
    shp = _lib.shape(F, Lv, Lt, D, heads, dtype)
    nbytes = lib.vc_block_stream_workspace_bytes(C.byref(shp))
    if nbytes == 0:
        _lib.check(lib.vc_block_shape_check(C.byref(shp)), "shape")
    ws = workspace(torch, nbytes)
    if outs is None:
        outs = [torch.empty((F, Lv, D), dtype=torch.float32).pin_memory() for _ in visuals]
    pin = prompt if _is_torch(prompt) else torch.from_numpy(np.ascontiguousarray(prompt, dtype=np.float32))
    pin = pin.contiguous().pin_memory() if not pin.is_pinned() else pin
    n = len(visuals)
    xs = (C.c_void_p * n)(*[v.data_ptr() for v in visuals])
    ys = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    streams = _HOST_STREAMS.setdefault("s", (torch.cuda.Stream(), torch.cuda.Stream()))
    _lib.check(lib.vc_block_forward_host_batched(C.byref(shp), _lib.ptr(db.packed), n, xs,
                                                 C.c_void_p(pin.data_ptr()), ys, _lib.ptr(ws), ws.numel(),
                                                 _lib.stream_ptr(torch), C.c_void_p(streams[0].cuda_stream),
                                                 C.c_void_p(streams[1].cuda_stream)), "host stream")
    return outs


_HOST_STREAMS: dict = {}


def _single_branch(params, slot, visual, text, heads, dtype):
    dim = visual.shape[2]
    z = BranchParams.zeros(dim)
    br = [z, z, z]
    br[slot] = params
    if text is None:
        text = np.zeros((1, 0, dim))
    return parallel_block_forward(BlockParams(*br), visual, text, heads, dtype=dtype)


def spatial_branch(params: BranchParams, visual, heads: int, *, dtype=None):
    """model.py:230-235 -- attention within each frame."""
    _check_visual(visual)
    return _single_branch(params, 0, visual, None, heads, dtype)


def temporal_branch(params: BranchParams, visual, heads: int, *, dtype=None):
    """model.py:238-244 -- attention across frames at each position."""
    _check_visual(visual)
    return _single_branch(params, 1, visual, None, heads, dtype)


def full_sequence_attention(params: BranchParams, text, visual, heads: int, *, dtype=None):
    """model.py:247-260 -- anchored text + all visual tokens; visual rows out."""
    _check_visual(visual, text)
    return _single_branch(params, 2, visual, text, heads, dtype)


def branch_attention(params: BranchParams, x, heads: int, *, dtype=None):
    """model.py:187-190 -- full branch on one resident [s, dim] sequence."""
    if x.ndim != 2:
        raise ValueError("branch_attention expects [s, dim]")
    out = spatial_branch(params, x[None], heads, dtype=dtype)
    return out[0]


def layer_norm(x, eps: float = 1e-5):
    """model.py:89-92 on the GPU (fp32). Only eps=1e-5 (the reference's) is built in."""
    if eps != 1e-5:
        raise ValueError("only the reference eps 1e-5 is supported")
    torch = _lib.require_cuda()
    as_numpy = not _is_torch(x)
    t = to_device_f32(torch, x)
    out = torch.empty_like(t)
    lib = _lib.load()
    D = t.shape[-1]
    _lib.check(lib.vc_layer_norm_f32(_lib.ptr(t), _lib.ptr(out), t.numel() // D, D,
                                     _lib.stream_ptr(torch)), "layer_norm")
    return out.double().cpu().numpy() if as_numpy else out


# ---------------------------------------------------------------------------
# The frame encoder (model.py:381-403) and forward noising (diffusion.py:77-84)
# ---------------------------------------------------------------------------

def encode_frames_device(torch, pixels_dev, spec: PatchSpec = PatchSpec(), schedule=None, t=None, noise_dev=None):
    """toy_vae_encode of every frame of a device clip [F, H, W, 3] fp32 ->
    latents [F, ceil(H/d), ceil(W/d), C] fp32, with q_sample (diffusion.py:77-84)
    fused when a schedule, t and noise are given (vc_vae_encode_frames)."""
    F, H, W, c = pixels_dev.shape
    if c != 3:
        raise ValueError(f"expected [h, w, 3] pixels, got {tuple(pixels_dev.shape[1:])}")
    gh, gw = spec.latent_hw(H, W)
    out = torch.empty((F, gh, gw, spec.latent_channels), dtype=torch.float32, device="cuda")
    sab, somab = 1.0, 0.0
    if noise_dev is not None:
        i = schedule._idx(int(t))
        sab, somab = math.sqrt(schedule.alpha_bars[i]), math.sqrt(schedule.one_minus_alpha_bars[i])
    lib = _lib.load()
    _lib.check(lib.vc_vae_encode_frames(_lib.ptr(pixels_dev), _lib.ptr(noise_dev), _lib.ptr(out), F, H, W,
                                        spec.vae_downsample, spec.latent_channels, sab, somab,
                                        _lib.stream_ptr(torch)), "vae encode")
    return out


def toy_vae_encode(frame, spec: PatchSpec = PatchSpec()):
    """model.py:381-403 -- [h, w, 3] pixels -> [ceil(h/8), ceil(w/8), C] latents
    (same signature and ValueError as the reference; on the GPU)."""
    if frame.ndim != 3 or frame.shape[2] != 3:
        raise ValueError(f"expected [h, w, 3] pixels, got {frame.shape}")
    torch = _lib.require_cuda()
    as_numpy = not _is_torch(frame)
    px = to_device_f32(torch, frame)[None]
    out = encode_frames_device(torch, px, spec)[0]
    return out.double().cpu().numpy() if as_numpy else out


# ---------------------------------------------------------------------------
# The toy denoiser (model.py:274-333)
# ---------------------------------------------------------------------------

@dataclass
class ToyDenoiser:
    spec: PatchSpec
    dim: int
    heads: int
    w_in: np.ndarray
    w_out: np.ndarray
    blocks: list = field(default_factory=list)

    @staticmethod
    def init(rng: SeededRng, spec: PatchSpec, dim: int, heads: int, depth: int) -> "ToyDenoiser":
        if dim % heads != 0:
            raise ValueError(f"dim {dim} not divisible by {heads} heads")
        pd = spec.patch * spec.patch * spec.latent_channels
        return ToyDenoiser(
            spec=spec, dim=dim, heads=heads,
            w_in=rng.split(1).normal((pd, dim)) / math.sqrt(pd),
            w_out=rng.split(2).normal((dim, pd)) / math.sqrt(dim),
            blocks=[BlockParams.init(rng.split(1000 + i), dim) for i in range(depth)],
        )

    @property
    def depth(self) -> int:
        return len(self.blocks)

    # -- device pieces ----------------------------------------------------------
    def _embed(self, torch, lat_dev, first_frame: int, t):
        F, h, w, c = lat_dev.shape
        if c != self.spec.latent_channels:
            raise ValueError(f"expected {self.spec.latent_channels} latent channels, got {c}")
        if self.dim % 2 != 0:
            raise ValueError(f"embedding dim must be even, got {self.dim}")
        p = self.spec.patch
        Lv = math.ceil(h / p) * math.ceil(w / p)
        w_in = to_device_f32(torch, self.w_in)
        x = torch.empty((F, Lv, self.dim), dtype=torch.float32, device="cuda")
        lib = _lib.load()
        _lib.check(lib.vc_embed_frames(_lib.ptr(lat_dev), _lib.ptr(w_in), _lib.ptr(x), F, first_frame,
                                       h, w, c, p, self.dim, float(t), _lib.stream_ptr(torch)), "embed")
        return x

    def _blocks(self, torch, x, prompt_dev, dtype):
        for blk in self.blocks:
            db = device_block(torch, blk, self.heads, dtype)
            block_forward_device(torch, db, x, prompt_dev, x, True)  # x = x + block(x)
        return x

    def head_states_device(self, latents, t, prompt, *, dtype=None):
        torch = _lib.require_cuda()
        dtype = _resolve_dtype(dtype)
        lat = to_device_f32(torch, latents)
        x = self._embed(torch, lat, 0, t)
        pr = to_device_f32(torch, prompt) if prompt.shape[0] > 0 else None
        return self._blocks(torch, x, pr, dtype)

    # -- reference API ---------------------------------------------------------------
    def embed_frame(self, latent, frame_index: int, t):
        """model.py:303-314 for one frame [h, w, c] -> [Lv, dim]."""
        torch = _lib.require_cuda()
        as_numpy = not _is_torch(latent)
        lat = to_device_f32(torch, latent)[None]
        x = self._embed(torch, lat, int(frame_index), t)[0]
        return x.double().cpu().numpy() if as_numpy else x

    def head_states(self, latents, t, prompt, *, dtype=None):
        """model.py:316-325 -- embed, then x = x + block(x) per block."""
        as_numpy = not _is_torch(latents)
        x = self.head_states_device(latents, t, prompt, dtype=dtype)
        return x.double().cpu().numpy() if as_numpy else x

    def denoise_step(self, latents, t, prompt, schedule, injected_noise=None, *, dtype=None):
        """One full sampling step x_t -> x_{t-1}: forward (model.py:327-333)
        with the reference's reverse_step (diffusion.py:95-116) fused into the
        unembed kernel (vc_unembed_reverse_step). At t == 1 or without
        injected noise the step returns the mean, as the reference does.
        Returns (x_prev, eps)."""
        torch = _lib.require_cuda()
        as_numpy = not _is_torch(latents)
        F, h, w, c = latents.shape
        coef_eps, inv_sqrt_alpha, sqrt_beta = schedule.reverse_coefficients(int(t))
        xt = to_device_f32(torch, latents)
        x = self.head_states_device(xt, t, prompt, dtype=dtype)
        w_out = to_device_f32(torch, self.w_out)
        eps = torch.empty((F, h, w, c), dtype=torch.float32, device="cuda")
        x_prev = torch.empty_like(eps)
        noise = None
        if injected_noise is not None and int(t) != 1:
            noise = to_device_f32(torch, injected_noise)
        lib = _lib.load()
        _lib.check(lib.vc_unembed_reverse_step(_lib.ptr(x), _lib.ptr(w_out), _lib.ptr(xt), _lib.ptr(noise),
                                               _lib.ptr(eps), _lib.ptr(x_prev), F, h, w, c, self.spec.patch,
                                               self.dim, float(coef_eps), float(inv_sqrt_alpha),
                                               float(sqrt_beta), _lib.stream_ptr(torch)), "denoise step")
        if as_numpy:
            return x_prev.double().cpu().numpy(), eps.double().cpu().numpy()
        return x_prev, eps

    def forward(self, latents, t, prompt, *, dtype=None):
        """model.py:327-333 -- predict the noise in a latent video [F, h, w, c]."""
        torch = _lib.require_cuda()
        as_numpy = not _is_torch(latents)
        F, h, w, c = latents.shape
        x = self.head_states_device(latents, t, prompt, dtype=dtype)
        w_out = to_device_f32(torch, self.w_out)
        eps = torch.empty((F, h, w, c), dtype=torch.float32, device="cuda")
        lib = _lib.load()
        _lib.check(lib.vc_unembed_frames(_lib.ptr(x), _lib.ptr(w_out), _lib.ptr(eps), F, h, w, c,
                                         self.spec.patch, self.dim, _lib.stream_ptr(torch)), "unembed")
        return eps.double().cpu().numpy() if as_numpy else eps

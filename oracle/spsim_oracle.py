"""CPU oracle for the parallel MM-DiT block forward -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference `spsim` hot path
(arXiv 2501.08453 / Vchitect-2.0 parallel multimodal diffusion block). It is
the *checker*: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it. The product package
(`paper_2501_08453_b200`) never imports it and has no CPU fallback.

Parity is pinned: `tests/golden/make_golden.py` ran the unmodified reference
(imported from /root/reference/pkg/src in the build container) and committed
its outputs under `tests/golden/`; `tests/test_oracle_golden.py` checks this
restatement against them (bitwise for integers, 1e-12 for floats).

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/spsim/). The restatement is vectorised (batched
einsum over frames / positions / heads) instead of the reference's Python
loops; the arithmetic per output element is the same.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------------------
# numerics.py
# ---------------------------------------------------------------------------

class SeededRng:
    """numerics.py:38-69 -- Philox counter RNG, substreams by seed XOR tag."""

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


def softmax_rows(x: np.ndarray) -> np.ndarray:
    """numerics.py:80-84 -- max-shifted softmax over the last axis."""
    e = np.exp(x - np.max(x, axis=-1, keepdims=True))
    return e / np.sum(e, axis=-1, keepdims=True)


def attention(q, k, v, heads: int, key_weight=None) -> np.ndarray:
    """numerics.py:87-107 -- per-head SDPA, heads = contiguous column slices.

    Batched over leading axes: q [..., s_q, d], k/v [..., s_k, d].
    `key_weight` (optional, [s_k]) multiplies each key's softmax weight; it
    is the oracle-side statement of key deduplication (a key present w
    times). The reference never passes it; tests use it to check the
    dedup identity against the replicated-key reference.
    """
    if q.shape[-1] % heads:
        raise ValueError(f"feature dim {q.shape[-1]} not divisible by {heads} heads")
    d = q.shape[-1]
    dh = d // heads
    # [..., s, h, dh] -> [..., h, s, dh]; batched BLAS matmuls per head
    qh = np.ascontiguousarray(np.swapaxes(q.reshape(q.shape[:-1] + (heads, dh)), -2, -3))
    kh = np.ascontiguousarray(np.swapaxes(k.reshape(k.shape[:-1] + (heads, dh)), -2, -3))
    vh = np.ascontiguousarray(np.swapaxes(v.reshape(v.shape[:-1] + (heads, dh)), -2, -3))
    s = (qh @ np.swapaxes(kh, -1, -2)) * (1.0 / np.sqrt(dh))
    if key_weight is not None:
        s = s + np.log(key_weight)
    o = softmax_rows(s) @ vh
    return np.ascontiguousarray(np.swapaxes(o, -2, -3)).reshape(q.shape)


# ---------------------------------------------------------------------------
# model.py
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class PatchSpec:
    """model.py:28-43."""
    vae_downsample: int = 8
    patch: int = 2
    latent_channels: int = 4

    def latent_hw(self, height, width):
        d = self.vae_downsample
        return (math.ceil(height / d), math.ceil(width / d))

    def tokens_per_frame(self, height, width):
        h, w = self.latent_hw(height, width)
        return math.ceil(h / self.patch) * math.ceil(w / self.patch)


def seq_len(frames, height, width, spec=PatchSpec()):
    """model.py:46-50."""
    if frames < 1 or height < 1 or width < 1:
        raise ValueError(f"bad clip shape ({frames}, {height}, {width})")
    return frames * spec.tokens_per_frame(height, width)


def patchify(latent, patch):
    """model.py:53-64 -- [h,w,c] -> [gh*gw, p*p*c], row-major grid, zero pad."""
    h, w, c = latent.shape
    gh, gw = -(-h // patch), -(-w // patch)
    buf = np.zeros((gh * patch, gw * patch, c))
    buf[:h, :w] = latent
    return buf.reshape(gh, patch, gw, patch, c).swapaxes(1, 2).reshape(gh * gw, patch * patch * c)


def unpatchify(tokens, h, w, c, patch):
    """model.py:67-76 -- inverse of patchify with crop."""
    gh, gw = -(-h // patch), -(-w // patch)
    if tokens.shape != (gh * gw, patch * patch * c):
        raise ValueError(f"token array {tokens.shape} does not match ({h}, {w}, {c}) at patch {patch}")
    return tokens.reshape(gh, gw, patch, patch, c).swapaxes(1, 2).reshape(gh * patch, gw * patch, c)[:h, :w]


def sinusoidal_embedding(position, dim):
    """model.py:79-86 -- [sin(pos*f_i) | cos(pos*f_i)], f_i = 10000^(-i/half)."""
    if dim % 2:
        raise ValueError(f"embedding dim must be even, got {dim}")
    half = dim // 2
    ang = np.asarray(position, dtype=np.float64)[..., None] * np.exp(
        -math.log(10000.0) * np.arange(half) / half)
    return np.concatenate([np.sin(ang), np.cos(ang)], axis=-1)


def layer_norm(x, eps=1e-5):
    """model.py:89-92 -- biased variance, no affine."""
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps)


def anchor_text(prompt, frames):
    """model.py:126-130."""
    if prompt.ndim != 2:
        raise ValueError("prompt must be [len, dim]")
    return np.repeat(prompt[None], frames, axis=0)


def interleave_checkerboard(text, visual):
    """model.py:133-140 -- [t0 v0 t1 v1 ...]."""
    return np.concatenate([text, visual], axis=1).reshape(-1, text.shape[-1])


def deinterleave_visual(seq, frames, text_len, visual_len):
    """model.py:143-154."""
    stride = text_len + visual_len
    if seq.shape[0] != frames * stride:
        raise ValueError("sequence does not tile")
    return seq.reshape(frames, stride, -1)[:, text_len:].copy()


@dataclass
class BranchParams:
    """model.py:157-178 -- draw order gamma, beta, wq, wk, wv, wo."""
    gamma: np.ndarray
    beta: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray

    @staticmethod
    def init(rng, dim):
        s = 1.0 / math.sqrt(dim)
        gamma = 1.0 + 0.02 * rng.normal(dim)
        beta = 0.02 * rng.normal(dim)
        wq = s * rng.normal((dim, dim))
        wk = s * rng.normal((dim, dim))
        wv = s * rng.normal((dim, dim))
        wo = s * rng.normal((dim, dim))
        return BranchParams(gamma, beta, wq, wk, wv, wo)


@dataclass
class BlockParams:
    """model.py:193-205 -- branch streams split(101/202/303)."""
    spatial: BranchParams
    temporal: BranchParams
    fullseq: BranchParams

    @staticmethod
    def init(rng, dim):
        return BlockParams(BranchParams.init(rng.split(101), dim),
                           BranchParams.init(rng.split(202), dim),
                           BranchParams.init(rng.split(303), dim))


def branch_qkv(p, x):
    """model.py:181-184."""
    n = layer_norm(x) * p.gamma + p.beta
    return n @ p.wq, n @ p.wk, n @ p.wv


def branch_attention(p, x, heads, key_weight=None):
    """model.py:187-190 (batched over leading axes)."""
    q, k, v = branch_qkv(p, x)
    return attention(q, k, v, heads, key_weight) @ p.wo


def spatial_branch(p, visual, heads):
    """model.py:230-235 -- one sequence per frame."""
    return branch_attention(p, visual, heads)


def temporal_branch(p, visual, heads):
    """model.py:238-244 -- one sequence per spatial position (transpose)."""
    return branch_attention(p, visual.transpose(1, 0, 2), heads).transpose(1, 0, 2)


def full_sequence_attention(p, text, visual, heads):
    """model.py:247-260 -- anchored text[0], checkerboard, visual rows only."""
    frames = visual.shape[0]
    seq = interleave_checkerboard(anchor_text(text[0], frames), visual)
    out = branch_attention(p, seq, heads)
    return deinterleave_visual(out, frames, text.shape[1], visual.shape[1])


def full_sequence_attention_dedup(p, text, visual, heads):
    """Same result as full_sequence_attention with the F anchored text copies
    collapsed to one key set of weight F (key/value permutation invariance,
    tests/test_numerics.py:131-140 in the reference). Only visual queries are
    evaluated. This is the algorithm the CUDA path implements; the tests
    check it equals full_sequence_attention."""
    frames, lv, d = visual.shape
    lt = text.shape[1]
    q, _, _ = branch_qkv(p, visual.reshape(-1, d))
    _, kt, vt = branch_qkv(p, text[0])
    _, kv, vv = branch_qkv(p, visual.reshape(-1, d))
    k = np.concatenate([kt, kv])
    v = np.concatenate([vt, vv])
    w = np.concatenate([np.full(lt, float(frames)), np.ones(frames * lv)])
    return (attention(q, k, v, heads, w) @ p.wo).reshape(frames, lv, d)


def parallel_block_forward(block, visual, text, heads):
    """model.py:263-271 -- spatial + temporal + fullseq, no residual."""
    return (spatial_branch(block.spatial, visual, heads)
            + temporal_branch(block.temporal, visual, heads)
            + full_sequence_attention(block.fullseq, text, visual, heads))


def _rows_attention(q, k, v, heads, chunk=32):
    """attention() for a few query rows against many keys, query-chunked so
    the [rows, keys] scores of all heads stay small (numerics.py:87-107)."""
    out = np.empty_like(q)
    for i in range(0, q.shape[0], chunk):
        out[i:i + chunk] = attention(q[i:i + chunk], k, v, heads)
    return out


def parallel_block_rows(block, visual, text, heads, f_idx, l_idx):
    """Rows (f_idx[i], l_idx[i]) of each branch of parallel_block_forward
    (model.py:263-271), computed for just those query rows: every key and
    value the rows attend to is projected (all Lv rows of a sampled frame for
    the spatial branch, model.py:230-235; all F frames of a sampled position
    for the temporal branch, model.py:238-244; the whole anchored
    checkerboard sequence, F literal copies of text[0] included, for the
    full-sequence branch, model.py:247-260), queries and the O projection
    only for the sampled rows. Returns {"spatial", "temporal", "fullseq",
    "block"}: [n, D] each. Same arithmetic per row as the full forward, so it
    is checked against parallel_block_forward on small shapes
    (tests/test_oracle_golden.py) and used at the full BASELINE shapes where
    the full fp64 forward does not fit a test's time budget."""
    f_idx = np.asarray(f_idx, dtype=np.int64)
    l_idx = np.asarray(l_idx, dtype=np.int64)
    frames, lv, d = visual.shape
    n = f_idx.size
    out = {k: np.zeros((n, d)) for k in ("spatial", "temporal", "fullseq")}
    # spatial: one sequence per frame
    p = block.spatial
    for f in np.unique(f_idx):
        sel = np.nonzero(f_idx == f)[0]
        q, _, _ = branch_qkv(p, visual[f, l_idx[sel]])
        _, k, v = branch_qkv(p, visual[f])
        out["spatial"][sel] = _rows_attention(q, k, v, heads) @ p.wo
    # temporal: one sequence per spatial position
    p = block.temporal
    for pos in np.unique(l_idx):
        sel = np.nonzero(l_idx == pos)[0]
        q, _, _ = branch_qkv(p, visual[f_idx[sel], pos])
        _, k, v = branch_qkv(p, visual[:, pos])
        out["temporal"][sel] = _rows_attention(q, k, v, heads) @ p.wo
    # full sequence: [t0 v0 t1 v1 ...] with every text slot = text[0]
    p = block.fullseq
    lt = text.shape[1]
    _, kt, vt = branch_qkv(p, text[0])
    kv = np.empty((frames, lv, d))
    vv = np.empty((frames, lv, d))
    for f in range(frames):  # frame by frame: the whole clip at once doubles the peak memory
        _, kv[f], vv[f] = branch_qkv(p, visual[f])
    k = np.concatenate([np.broadcast_to(kt, (frames, lt, d)), kv], axis=1).reshape(-1, d)
    del kv
    v = np.concatenate([np.broadcast_to(vt, (frames, lt, d)), vv], axis=1).reshape(-1, d)
    del vv
    q, _, _ = branch_qkv(p, visual[f_idx, l_idx])
    out["fullseq"] = _rows_attention(q, k, v, heads) @ p.wo
    out["block"] = out["spatial"] + out["temporal"] + out["fullseq"]
    return out


def _channel_mix(channels):
    """model.py:399-403 -- fixed [3, C] cosine projection."""
    j = np.arange(3)[:, None]
    i = np.arange(channels)[None, :]
    return math.sqrt(2.0 / 3.0) * np.cos(math.pi * (2 * j + 1) * i / 6.0)


def toy_vae_encode(frame, spec=PatchSpec()):
    """model.py:381-396 -- zero-pad to a multiple of d, d x d block mean, channel mix."""
    d = spec.vae_downsample
    h, w, _ = frame.shape
    gh, gw = math.ceil(h / d), math.ceil(w / d)
    padded = np.zeros((gh * d, gw * d, 3))
    padded[:h, :w] = frame
    return padded.reshape(gh, d, gw, d, 3).mean(axis=(1, 3)) @ _channel_mix(spec.latent_channels)


@dataclass
class ToyDenoiser:
    """model.py:274-333."""
    spec: PatchSpec
    dim: int
    heads: int
    w_in: np.ndarray
    w_out: np.ndarray
    blocks: list = field(default_factory=list)

    @staticmethod
    def init(rng, spec, dim, heads, depth):
        if dim % heads:
            raise ValueError(f"dim {dim} not divisible by {heads} heads")
        pd = spec.patch * spec.patch * spec.latent_channels
        return ToyDenoiser(spec, dim, heads,
                           rng.split(1).normal((pd, dim)) / math.sqrt(pd),
                           rng.split(2).normal((dim, pd)) / math.sqrt(dim),
                           [BlockParams.init(rng.split(1000 + i), dim) for i in range(depth)])

    def embed_frame(self, latent, frame_index, t):
        """model.py:303-314 -- patchify@w_in + sin(global index) + sin(t)."""
        tokens = patchify(latent, self.spec.patch) @ self.w_in
        n = tokens.shape[0]
        tokens = tokens + sinusoidal_embedding(frame_index * n + np.arange(n, dtype=np.float64), self.dim)
        return tokens + sinusoidal_embedding(float(t), self.dim)

    def head_states(self, latents, t, prompt):
        """model.py:316-325."""
        frames = latents.shape[0]
        x = np.stack([self.embed_frame(latents[f], f, t) for f in range(frames)])
        text = anchor_text(prompt, frames)
        for b in self.blocks:
            x = x + parallel_block_forward(b, x, text, self.heads)
        return x

    def forward(self, latents, t, prompt):
        """model.py:327-333."""
        _, h, w, c = latents.shape
        x = self.head_states(latents, t, prompt)
        return np.stack([unpatchify(x[f] @ self.w_out, h, w, c, self.spec.patch)
                         for f in range(x.shape[0])])


# ---------------------------------------------------------------------------
# diffusion.py -- schedule and the ancestral reverse step
# ---------------------------------------------------------------------------

def make_linear_schedule(steps, beta_start=1e-4, beta_end=0.02):
    """diffusion.py:56-66 + NoiseSchedule diffusion.py:17-53 -> dict of arrays."""
    betas = (np.array([beta_start]) if steps == 1
             else np.linspace(beta_start, beta_end, steps, dtype=np.float64))
    alphas = 1.0 - betas
    abar = np.cumprod(alphas)
    return {"betas": betas, "alphas": alphas, "alpha_bars": abar, "omab": 1.0 - abar}


def q_sample(schedule, x0, t, noise):
    """diffusion.py:77-84 -- x_t in closed form from clean data."""
    i = t - 1
    return np.sqrt(schedule["alpha_bars"][i]) * x0 + np.sqrt(schedule["omab"][i]) * noise


def reverse_step(schedule, x_t, t, predicted_noise, injected_noise=None):
    """diffusion.py:95-116 -- x_t -> x_{t-1}; no noise at t == 1."""
    i = t - 1
    beta, alpha, omab = schedule["betas"][i], schedule["alphas"][i], schedule["omab"][i]
    mean = (x_t - (beta / np.sqrt(omab)) * predicted_noise) / np.sqrt(alpha)
    if t == 1 or injected_noise is None:
        return mean
    return mean + np.sqrt(beta) * injected_noise


# ---------------------------------------------------------------------------
# executor.py -- shard maps (integer, exact)
# ---------------------------------------------------------------------------

def contiguous_bounds(n, p):
    """executor.py:187-191 -- bounds[i] = i*n//p."""
    if p < 1:
        raise ValueError(f"cannot split into {p} parts")
    return [i * n // p for i in range(p + 1)]


def round_robin_frames(frames, p):
    """executor.py:194-196."""
    return [list(range(d, frames, p)) for d in range(p)]


def fused_equal_division(text_len, visual_len, p):
    """executor.py:199-213."""
    b = contiguous_bounds(text_len + visual_len, p)
    out = []
    for lo, hi in zip(b[:-1], b[1:]):
        t = max(0, min(text_len, hi) - min(text_len, lo))
        out.append((t, hi - lo - t))
    return out


def placement_division(text_len, visual_len, p, placement):
    """executor.py:216-229."""
    if placement == "separate":
        tb, vb = contiguous_bounds(text_len, p), contiguous_bounds(visual_len, p)
        return ([tb[i + 1] - tb[i] for i in range(p)], [vb[i + 1] - vb[i] for i in range(p)])
    if placement == "fused":
        parts = fused_equal_division(text_len, visual_len, p)
        return [t for t, _ in parts], [v for _, v in parts]
    raise ValueError(f"unknown text placement {placement!r}")


def prefix_bounds(counts):
    """executor.py:241-245."""
    return [0] + list(np.cumsum(counts, dtype=np.int64).tolist())


def fullseq_global_order(frames, text_len, visual_len, p):
    """executor.py:598-617 + :349-370 -- the global index keys each device's
    fullseq chunks carry (spatial axis, separate placement), and the stable
    argsort that assembles the sequence. Returns (idx_by_dev, order)."""
    tc, vc = placement_division(text_len, visual_len, p, "separate")
    tb, vb = prefix_bounds(tc), prefix_bounds(vc)
    stride = text_len + visual_len
    idx_by_dev = []
    for dev in range(p):
        parts = []
        for f in range(frames):
            base = f * stride
            if tb[dev + 1] > tb[dev]:
                parts.append(np.arange(base + tb[dev], base + tb[dev + 1]))
            parts.append(np.arange(base + text_len + vb[dev], base + text_len + vb[dev + 1]))
        idx_by_dev.append(np.concatenate(parts) if parts else np.zeros(0, np.int64))
    order = np.argsort(np.concatenate(idx_by_dev), kind="stable")
    return idx_by_dev, order


def comm_plan(frames, text_len, visual_len, dim, heads, depth, p, attention="head_parallel", bpe=8,
              placement="intra"):
    """executor.py:721-773 -- the collective schedule run_sp_iteration logs
    (spatial shard axis, separate text placement, one node): rows of
    (stage, collective, group_size, placement, bytes_per_device)
    (CommEvent.key, executor.py:100-108). Pinned by the reference
    executor's own log (tests/golden sp_p{P}_comm)."""
    if p <= 1:
        return []
    tcounts, vcounts = placement_division(text_len, visual_len, p, "separate")
    fsizes = [len(fs) for fs in round_robin_frames(frames, p)]
    col_width = dim // p if attention == "head_parallel" else dim
    rows = [("reshard", "alltoall", p, placement, float(max(fsizes) * visual_len * dim * bpe))]

    def branch(stage, rows_per_dev, needed_rows):
        if attention == "head_parallel":
            rows.append((stage, "alltoall", p, placement, float(3 * max(rows_per_dev) * dim * bpe)))
            rows.append((stage, "alltoall", p, placement, float(needed_rows * col_width * bpe)))
        else:
            rows.append((stage, "allgather", p, placement, float(2 * max(rows_per_dev) * dim * bpe)))

    for bi in range(depth):
        branch(f"block{bi}.spatial", [frames * v for v in vcounts], frames * visual_len)
        branch(f"block{bi}.fullseq", [frames * (t + v) for t, v in zip(tcounts, vcounts)], frames * visual_len)
    rows.append(("gather", "allgather", p, placement, float(max(frames * v for v in vcounts) * dim * bpe)))
    return rows


def head_parallel_block(block, visual, text, heads, p):
    """executor.py:561-626 stage 3 (spatial axis, head-parallel, separate
    text placement) for one block, simulated on p logical devices in one
    process. Returns the per-device update arrays [F, vcount_r, D] (no
    residual). Used by the tests to check the multi-process exchange logic.
    """
    frames, lv, d = visual.shape
    if heads % p:
        raise ValueError("head-parallel attention needs sp_size | heads")
    _, vc = placement_division(text.shape[1], lv, p, "separate")
    vb = prefix_bounds(vc)
    full = parallel_block_forward(block, visual, text, heads)
    return [full[:, vb[r]:vb[r + 1]] for r in range(p)]

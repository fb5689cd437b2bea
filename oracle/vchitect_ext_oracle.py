"""CPU oracle for the north-star extensions of the block -- TEST INFRASTRUCTURE
ONLY, PARITY UNPINNED.

BASELINE.json's north_star names pieces of the Vchitect-2.0 block that the
reference `spsim` does not have (SURVEY.md §8 "a-ext"): QK-RMSNorm and 3D RoPE
on the spatial / full-sequence Q and K, AdaLN timestep modulation
(shift / scale / gate) and the gated FFN. There is no reference code, test or
golden vector for them, so this float64 numpy module *defines* the semantics
the CUDA path (`paper_2501_08453_b200.vchitect`) is checked against; the
reference-semantics block inside it is the pinned oracle
(`spsim_oracle.parallel_block_forward`, model.py:263-271). Only `tests/` may
import this module.

Semantics (x [F, Lv, D] visual tokens, prompt [Lt, D], integer timestep t):

    mod = silu(sinusoidal_embedding(t, D)) @ w_ada + b_ada          [6D]
        -> shift_msa, scale_msa, gate_msa, shift_mlp, scale_mlp, gate_mlp
    a    = LN(x) * (1 + scale_msa) + shift_msa    (prompt rows likewise)
    per branch n = a * gamma + beta; q, k, v = n @ wq, n @ wk, n @ wv
      spatial / full-sequence: per head q_h <- rope(rms(q_h) * q_norm),
      k_h <- rope(rms(k_h) * k_norm); rms(u) = u / sqrt(mean(u^2) + 1e-6)
      over the dh real dims; the temporal branch is unchanged
    attn = spatial + temporal + fullseq        (model.py:267-271 order)
    h    = x + gate_msa * attn
    n2   = LN(h) * (1 + scale_mlp) + shift_mlp
    y    = h + gate_mlp * (gelu_tanh(n2 @ w1 + b1) @ w2 + b2)

3D RoPE: visual token l of frame f sits at (f, l // gw, l % gw) on the
(gh, gw) patch grid. The dh/2 rotation pairs (2i, 2i+1) split into
n_t = P - 2 (P // 3) temporal, then P // 3 row and P // 3 column pairs
(P = dh / 2); pair j of an axis with n_a pairs turns by pos * base^(-j / n_a),
base 1e4: (u0, u1) -> (u0 c - u1 s, u0 s + u1 c). Text tokens carry no
position (identity rotation): the F anchored copies stay identical, so the
full-sequence key deduplication (+ log F on the text logits) stays exact.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from oracle import spsim_oracle as O

RMS_EPS = 1e-6
ROPE_BASE = 10000.0


def silu(x):
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def rope_split(dh):
    if dh % 2:
        raise ValueError(f"3D RoPE needs an even head dim, got {dh}")
    p = dh // 2
    ny = nx = p // 3
    return p - ny - nx, ny, nx


def rope_angles(dh, pos_t, pos_y, pos_x):
    """Angles [..., dh/2] of the pairs for positions pos_* (same shapes)."""
    nt, ny, nx = rope_split(dh)
    parts = []
    for pos, n in ((pos_t, nt), (pos_y, ny), (pos_x, nx)):
        theta = ROPE_BASE ** (-np.arange(n, dtype=np.float64) / max(n, 1))
        parts.append(np.asarray(pos, dtype=np.float64)[..., None] * theta)
    return np.concatenate(parts, axis=-1)


def apply_rope(u, heads, ang):
    """u [rows, H*dh], ang [rows, dh/2] (None: identity)."""
    if ang is None:
        return u
    rows, d = u.shape
    dh = d // heads
    r = u.reshape(rows, heads, dh // 2, 2)
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    out = np.empty_like(r)
    out[..., 0] = r[..., 0] * c - r[..., 1] * s
    out[..., 1] = r[..., 0] * s + r[..., 1] * c
    return out.reshape(rows, d)


def rms_heads(u, heads, w):
    rows, d = u.shape
    r = u.reshape(rows, heads, d // heads)
    r = r / np.sqrt((r * r).mean(axis=-1, keepdims=True) + RMS_EPS) * w
    return r.reshape(rows, d)


@dataclass
class VchitectExtParams:
    """Draw order from rng.split(404): w_ada, b_ada, q_norm[2, dh],
    k_norm[2, dh] (rows: spatial, full sequence), w1, b1, w2, b2."""
    block: O.BlockParams
    w_ada: np.ndarray   # [D, 6D]
    b_ada: np.ndarray   # [6D]
    q_norm: np.ndarray  # [2, dh]
    k_norm: np.ndarray  # [2, dh]
    w1: np.ndarray      # [D, Dff]
    b1: np.ndarray      # [Dff]
    w2: np.ndarray      # [Dff, D]
    b2: np.ndarray      # [D]

    @staticmethod
    def init(rng, dim, heads, mlp_ratio=2.0):
        dh = dim // heads
        dff = int(round(dim * mlp_ratio))
        block = O.BlockParams.init(rng.split(1000), dim)
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


def modulation(p, t, dim):
    mod = silu(O.sinusoidal_embedding(float(t), dim)) @ p.w_ada + p.b_ada
    return mod.reshape(6, dim)


def _qkv(bp, a):
    n = a * bp.gamma + bp.beta
    return n @ bp.wq, n @ bp.wk, n @ bp.wv


def vchitect_block_forward(p, visual, prompt, heads, t, grid):
    """The extended block on [F, Lv, D] visual tokens; returns y [F, Lv, D]
    (residuals included, unlike the reference block)."""
    F, Lv, D = visual.shape
    Lt = prompt.shape[0]
    gh, gw = grid
    if gh * gw != Lv:
        raise ValueError(f"grid {gh}x{gw} does not hold {Lv} tokens")
    dh = D // heads
    sh1, sc1, g1, sh2, sc2, g2 = modulation(p, t, D)
    a = O.layer_norm(visual) * (1 + sc1) + sh1
    at = O.layer_norm(prompt) * (1 + sc1) + sh1
    fi, li = np.meshgrid(np.arange(F), np.arange(Lv), indexing="ij")
    ang = rope_angles(dh, fi, li // gw, li % gw).reshape(F * Lv, -1)

    # spatial: one sequence per frame, rotated + normalised Q/K
    bp = p.block.spatial
    q, k, v = _qkv(bp, a.reshape(F * Lv, D))
    q = apply_rope(rms_heads(q, heads, p.q_norm[0]), heads, ang)
    k = apply_rope(rms_heads(k, heads, p.k_norm[0]), heads, ang)
    sp = O.attention(q.reshape(F, Lv, D), k.reshape(F, Lv, D), v.reshape(F, Lv, D), heads)
    sp = sp.reshape(F * Lv, D) @ bp.wo

    # temporal: unchanged branch (one sequence per spatial position)
    bp = p.block.temporal
    q, k, v = _qkv(bp, a.transpose(1, 0, 2))
    tm = (O.attention(q, k, v, heads) @ bp.wo).transpose(1, 0, 2).reshape(F * Lv, D)

    # full sequence: the literal checkerboard [t0 v0 t1 v1 ...] (model.py:247-260)
    bp = p.block.fullseq
    qv, kv, vv = _qkv(bp, a.reshape(F * Lv, D))
    _, kt, vt = _qkv(bp, at)
    qv = apply_rope(rms_heads(qv, heads, p.q_norm[1]), heads, ang)
    kv = apply_rope(rms_heads(kv, heads, p.k_norm[1]), heads, ang)
    kt = rms_heads(kt, heads, p.k_norm[1])
    ks, vs = [], []
    for f in range(F):
        ks += [kt, kv[f * Lv:(f + 1) * Lv]]
        vs += [vt, vv[f * Lv:(f + 1) * Lv]]
    fs = O.attention(qv, np.concatenate(ks), np.concatenate(vs), heads) @ bp.wo

    h = visual.reshape(F * Lv, D) + g1 * (sp + tm + fs)
    n2 = O.layer_norm(h) * (1 + sc2) + sh2
    y = h + g2 * (gelu_tanh(n2 @ p.w1 + p.b1) @ p.w2 + p.b2)
    return y.reshape(F, Lv, D)

"""CPU checks of the north-star extensions (PARITY UNPINNED: no reference
counterpart, oracle/vchitect_ext_oracle.py defines the semantics): the
oracle's own identities, the package's parameter init against the oracle's,
and the C-ABI size / shape queries (no compute calls without a GPU)."""
import ctypes as C

import numpy as np
import pytest

from oracle import spsim_oracle as O
from oracle import vchitect_ext_oracle as X
from paper_2501_08453_b200 import _lib


def test_rope_split_and_rotation_is_orthogonal():
    assert X.rope_split(66) == (11, 11, 11)
    assert X.rope_split(128) == (22, 21, 21)
    assert X.rope_split(64) == (12, 10, 10)
    r = np.random.default_rng(0)
    u = r.standard_normal((7, 3 * 66))
    ang = X.rope_angles(66, r.integers(0, 9, 7), r.integers(0, 5, 7), r.integers(0, 6, 7))
    v = X.apply_rope(u, 3, ang)
    # rotations keep every head's norm and pair norms
    np.testing.assert_allclose(np.linalg.norm(v.reshape(7, 3, 33, 2), axis=-1),
                               np.linalg.norm(u.reshape(7, 3, 33, 2), axis=-1), rtol=1e-12)


def test_rope_is_relative():
    # q(p1) . k(p2) depends only on p1 - p2 (per axis)
    r = np.random.default_rng(1)
    q, k = r.standard_normal((1, 66)), r.standard_normal((1, 66))

    def dot(p1, p2):
        a1 = X.rope_angles(66, *[np.array([c]) for c in p1])
        a2 = X.rope_angles(66, *[np.array([c]) for c in p2])
        return float((X.apply_rope(q, 1, a1) @ X.apply_rope(k, 1, a2).T)[0, 0])

    assert abs(dot((3, 2, 5), (1, 1, 1)) - dot((5, 4, 9), (3, 3, 5))) < 1e-9


def _dedup_fullseq(p, a_vis, a_txt, heads, ang, F):
    """Full-sequence branch with the F text copies collapsed to one key set
    of weight F -- what the CUDA path computes."""
    bp = p.block.fullseq
    qv, kv, vv = X._qkv(bp, a_vis)
    _, kt, vt = X._qkv(bp, a_txt)
    qv = X.apply_rope(X.rms_heads(qv, heads, p.q_norm[1]), heads, ang)
    kv = X.apply_rope(X.rms_heads(kv, heads, p.k_norm[1]), heads, ang)
    kt = X.rms_heads(kt, heads, p.k_norm[1])
    w = np.concatenate([np.full(kt.shape[0], float(F)), np.ones(kv.shape[0])])
    return O.attention(qv, np.concatenate([kt, kv]), np.concatenate([vt, vv]), heads, w) @ bp.wo


def test_text_dedup_stays_exact_under_rope():
    # unrotated text keys keep the F anchored copies identical, so the
    # log-F deduplication the kernels use equals the literal checkerboard
    F, gh, gw, Lt, D, H = 3, 2, 3, 4, 24, 2
    p = X.VchitectExtParams.init(O.SeededRng(5), D, H)
    r = np.random.default_rng(2)
    x = r.standard_normal((F, gh * gw, D))
    prompt = r.standard_normal((Lt, D))
    y = X.vchitect_block_forward(p, x, prompt, H, 17, (gh, gw))
    # rebuild y with the dedup full-sequence branch
    sh1, sc1, g1, sh2, sc2, g2 = X.modulation(p, 17, D)
    a = O.layer_norm(x) * (1 + sc1) + sh1
    at = O.layer_norm(prompt) * (1 + sc1) + sh1
    fi, li = np.meshgrid(np.arange(F), np.arange(gh * gw), indexing="ij")
    ang = X.rope_angles(D // H, fi, li // gw, li % gw).reshape(F * gh * gw, -1)
    bp = p.block.spatial
    q, k, v = X._qkv(bp, a.reshape(-1, D))
    q = X.apply_rope(X.rms_heads(q, H, p.q_norm[0]), H, ang)
    k = X.apply_rope(X.rms_heads(k, H, p.k_norm[0]), H, ang)
    sp = O.attention(q.reshape(F, -1, D), k.reshape(F, -1, D), v.reshape(F, -1, D), H).reshape(-1, D) @ bp.wo
    bp = p.block.temporal
    q, k, v = X._qkv(bp, a.transpose(1, 0, 2))
    tm = (O.attention(q, k, v, H) @ bp.wo).transpose(1, 0, 2).reshape(-1, D)
    fs = _dedup_fullseq(p, a.reshape(-1, D), at, H, ang, F)
    h = x.reshape(-1, D) + g1 * (sp + tm + fs)
    n2 = O.layer_norm(h) * (1 + sc2) + sh2
    y2 = h + g2 * (X.gelu_tanh(n2 @ p.w1 + p.b1) @ p.w2 + p.b2)
    np.testing.assert_allclose(y.reshape(-1, D), y2, rtol=1e-10, atol=1e-10)


def test_zero_modulation_gates_are_identity():
    F, gh, gw, Lt, D, H = 2, 2, 2, 3, 16, 2
    p = X.VchitectExtParams.init(O.SeededRng(1), D, H)
    p.w_ada[:] = 0.0
    p.b_ada[:] = 0.0  # gates 0 -> y = x exactly
    x = np.random.default_rng(3).standard_normal((F, gh * gw, D))
    y = X.vchitect_block_forward(p, x, np.ones((Lt, D)), H, 5, (gh, gw))
    np.testing.assert_array_equal(y, x)


def test_package_init_matches_oracle_init():
    from paper_2501_08453_b200 import SeededRng
    from paper_2501_08453_b200.vchitect import VchitectExtParams
    a = VchitectExtParams.init(SeededRng(9), 48, 4, mlp_ratio=2.0)
    b = X.VchitectExtParams.init(O.SeededRng(9), 48, 4, mlp_ratio=2.0)
    for u, v in zip(a.ext_arrays(), (b.w_ada, b.b_ada, b.q_norm, b.k_norm, b.w1, b.b1, b.w2, b.b2)):
        np.testing.assert_array_equal(u, v)
    np.testing.assert_array_equal(a.block.fullseq.wo, b.block.fullseq.wo)


def _ext(F, Lv, Lt, D, H, grid, dff):
    from paper_2501_08453_b200.vchitect import ext_shape
    return ext_shape(F, Lv, Lt, D, H, grid, dff)


def test_ext_size_queries():
    lib = _lib.load()
    D, H, dff = 1584, 24, 3168
    s = _ext(16, 1350, 256, D, H, (30, 45), dff)
    dh = D // H
    assert lib.vc_ext_raw_weight_floats(C.byref(s)) == D * 6 * D + 6 * D + 4 * dh + 2 * D * dff + dff + D
    assert lib.vc_ext_packed_weight_bytes(C.byref(s)) >= D * 6 * D * 4 + 2 * D * dff * 2
    blk = _lib.shape(16, 1350, 256, D, H, "bf16")
    assert lib.vc_ext_workspace_bytes(C.byref(s)) > lib.vc_block_workspace_bytes(C.byref(blk))
    assert lib.vc_ext_block_launches(C.byref(s)) == 13


@pytest.mark.parametrize("args,msg", [
    ((2, 48, 4, 256, 4, (6, 7), 512), b"does not hold"),       # grid != Lv
    ((2, 48, 4, 256, 4, (6, 8), 500), b"multiple of 8"),       # ffn width
    ((2, 48, 4, 264, 8, (6, 8), 512), b"even head dim"),       # dh 33
])
def test_ext_shape_errors(args, msg):
    lib = _lib.load()
    s = _ext(*args)
    assert lib.vc_ext_raw_weight_floats(C.byref(s)) == 0
    assert msg in lib.vc_last_error()
    fp32 = _lib.ExtShape(_lib.shape(2, 48, 4, 256, 4, "fp32"), 6, 8, 512)
    assert lib.vc_ext_workspace_bytes(C.byref(fp32)) == 0
    assert b"bf16" in lib.vc_last_error()

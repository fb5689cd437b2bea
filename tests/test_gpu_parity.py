"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the pinned oracle, at the north-star tolerances:

  fp32 path : normwise max|y - ref| / max|ref| <= 1e-4
  bf16 path : relative L2 ||y - ref|| / ||ref|| <= 2e-2  (pre-residual block output)

Inputs come from SeededRng with the seeding convention of
tests/golden/make_golden.py.
"""
import numpy as np
import pytest

from oracle import spsim_oracle as O

pytestmark = pytest.mark.gpu

G = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "golden.npz"))
DATA_TAG = 1 << 20
FP32_TOL = 1e-4
BF16_TOL = 2e-2

BLOCK_CASES = [
    ("blk_tiny", 4, 64, 32, 256, 4),
    ("blk_small", 3, 5, 2, 12, 4),
    ("blk_odd", 2, 7, 3, 18, 3),
    ("blk_dh66", 2, 24, 8, 132, 2),
]


def normwise(y, ref):
    return float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))


def rel_l2(y, ref):
    return float(np.linalg.norm(y - ref) / np.linalg.norm(ref))


@pytest.fixture(scope="module")
def vc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2501_08453_b200 as vc
    return vc


def block_case(vc, name, F, Lv, Lt, D):
    seed = sum(map(ord, name))
    blk = vc.BlockParams.init(vc.SeededRng(seed).split(1000), D)
    data = vc.SeededRng(seed).split(DATA_TAG)
    x = data.split(1).normal((F, Lv, D))
    prompt = data.split(2).normal((Lt, D))
    return blk, x, prompt


def test_attention_known_answers(vc):
    q, k, v = G["attn_q"], G["attn_k"], G["attn_v"]
    for h in (1, 2, 4):
        got = vc.attention(q, k, v, h)
        assert normwise(got, G[f"attn_out_h{h}"]) < 1e-5
    # single key: output is v (reference tests/test_numerics.py:95-100)
    r = vc.SeededRng(8)
    q = r.normal((5, 4)); k1 = r.normal((1, 4)); v1 = r.normal((1, 4))
    np.testing.assert_allclose(vc.attention(q, k1, v1, 2), np.repeat(v1, 5, axis=0), atol=1e-6)
    with pytest.raises(ValueError):
        vc.attention(np.zeros((4, 6)), np.zeros((4, 6)), np.zeros((4, 6)), 4)


def test_attention_ragged_lengths_match_oracle(vc):
    r = vc.SeededRng(99)
    for sq, sk, d, h in ((1, 1, 8, 2), (33, 17, 64, 1), (100, 257, 132, 2), (7, 300, 256, 2)):
        q, k, v = r.normal((sq, d)), r.normal((sk, d)), r.normal((sk, d))
        assert normwise(vc.attention(q, k, v, h), O.attention(q, k, v, h)) < 1e-5


@pytest.mark.parametrize("case", BLOCK_CASES, ids=[c[0] for c in BLOCK_CASES])
def test_block_fp32_matches_reference(vc, case):
    name, F, Lv, Lt, D, H = case
    blk, x, prompt = block_case(vc, name, F, Lv, Lt, D)
    text = vc.anchor_text(prompt, F)
    got = vc.parallel_block_forward(blk, x, text, H, dtype="fp32")
    assert normwise(got, G[f"{name}_out"]) <= FP32_TOL
    assert normwise(vc.spatial_branch(blk.spatial, x, H), G[f"{name}_sp"]) <= FP32_TOL
    assert normwise(vc.temporal_branch(blk.temporal, x, H), G[f"{name}_tm"]) <= FP32_TOL
    assert normwise(vc.full_sequence_attention(blk.fullseq, text, x, H), G[f"{name}_fs"]) <= FP32_TOL


@pytest.mark.parametrize("case", [c for c in BLOCK_CASES if c[4] % 8 == 0], ids=lambda c: c[0])
def test_block_bf16_matches_reference(vc, case):
    name, F, Lv, Lt, D, H = case
    blk, x, prompt = block_case(vc, name, F, Lv, Lt, D)
    got = vc.parallel_block_forward(blk, x, vc.anchor_text(prompt, F), H, dtype="bf16")
    assert rel_l2(got, G[f"{name}_out"]) <= BF16_TOL


def test_text_anchoring_ignores_later_frames(vc):
    # reference tests/test_model.py:152-163: garbage in text[1:] changes nothing
    # (fp32 on a 12-dim block; bf16 needs dim % 8 == 0, so a 64-dim one)
    for name, D, dt in (("blk_small", 12, "fp32"), ("anchor_bf16", 64, "bf16")):
        blk, x, prompt = block_case(vc, name, 3, 5, 2, D)
        clean = vc.anchor_text(prompt, 3)
        dirty = clean.copy()
        dirty[1:] = vc.SeededRng(5).normal((2, 2, D)) * 100
        a = vc.full_sequence_attention(blk.fullseq, clean, x, 4, dtype=dt)
        b = vc.full_sequence_attention(blk.fullseq, dirty, x, 4, dtype=dt)
        assert np.array_equal(a, b), dt


def test_spatial_frames_independent(vc):
    # reference tests/test_model.py:179-189
    r = vc.SeededRng(7)
    p = vc.BranchParams.init(r.split(3), 8)
    visual = r.normal((4, 5, 8))
    out = vc.spatial_branch(p, visual, 2)
    perm = np.array([2, 0, 3, 1])
    np.testing.assert_allclose(out[perm], vc.spatial_branch(p, visual[perm], 2), atol=1e-6)


def test_block_is_sum_of_branches(vc):
    # reference tests/test_model.py:203-214 (exact there; here all on one device, fp32)
    blk, x, prompt = block_case(vc, "blk_tiny", 4, 64, 32, 256)
    text = vc.anchor_text(prompt, 4)
    tot = vc.parallel_block_forward(blk, x, text, 4)
    parts = (vc.spatial_branch(blk.spatial, x, 4) + vc.temporal_branch(blk.temporal, x, 4)
             + vc.full_sequence_attention(blk.fullseq, text, x, 4))
    assert normwise(tot, parts) < 1e-5


def model_case(vc, name, seed, F, h, w, Lt, D, H, depth):
    model = vc.ToyDenoiser.init(vc.SeededRng(seed), vc.PatchSpec(8, 2, 4), D, H, depth)
    data = vc.SeededRng(seed).split(DATA_TAG)
    lat = data.split(1).normal((F, h, w, 4))
    prompt = data.split(2).normal((Lt, D))
    return model, lat, prompt


@pytest.mark.parametrize("case", [("cfg1", 2501, 4, 16, 16, 32, 256, 4, 2, 37),
                                  ("mdl_ragged", 7, 3, 5, 7, 3, 12, 6, 1, 11)], ids=lambda c: c[0])
def test_model_forward_fp32_config1(vc, case):
    name, seed, F, h, w, Lt, D, H, depth, t = case
    model, lat, prompt = model_case(vc, name, seed, F, h, w, Lt, D, H, depth)
    assert normwise(model.embed_frame(lat[0], 0, t), G[f"{name}_embed0"]) <= 1e-6
    assert normwise(model.head_states(lat, t, prompt), G[f"{name}_states"]) <= FP32_TOL
    assert normwise(model.forward(lat, t, prompt), G[f"{name}_out"]) <= FP32_TOL


def test_model_forward_bf16_config1(vc):
    model, lat, prompt = model_case(vc, "cfg1", 2501, 4, 16, 16, 32, 256, 4, 2)
    got = model.forward(lat, 37, prompt, dtype="bf16")
    assert rel_l2(got, G["cfg1_out"]) <= BF16_TOL


def test_denoise_step_fused_reverse_step(vc):
    # forward + reverse_step (diffusion.py:95-116) fused into the unembed,
    # against the reference's own step (golden), t = 37 with noise and t = 1
    from paper_2501_08453_b200.diffusion import make_linear_schedule
    model, lat, prompt = model_case(vc, "cfg1", 2501, 4, 16, 16, 32, 256, 4, 2)
    z = vc.SeededRng(2501).split(DATA_TAG).split(3).normal((4, 16, 16, 4))
    sched = make_linear_schedule(100)
    for t in (37, 1):
        x_prev, eps = model.denoise_step(lat, t, prompt, sched, z)
        assert normwise(x_prev, G[f"rev_t{t}"]) <= FP32_TOL
        assert normwise(eps, model.forward(lat, t, prompt)) <= 1e-6
    x16, _ = model.denoise_step(lat, 37, prompt, sched, z, dtype="bf16")
    assert rel_l2(x16, G["rev_t37"]) <= BF16_TOL


def test_weight_mutation_is_seen(vc):
    # reference tests/test_model.py:256-262 mutates w_out in place
    model, lat, prompt = model_case(vc, "cfg1", 2501, 4, 16, 16, 32, 256, 4, 2)
    a = model.forward(lat, 37, prompt)
    model.w_out *= 2.0
    b = model.forward(lat, 37, prompt)
    np.testing.assert_allclose(b, 2 * a, rtol=1e-5, atol=1e-6)
    model.blocks[0].fullseq.wo[:] = 0.0
    c = model.forward(lat, 37, prompt)
    assert not np.allclose(c, b)


def test_device_weight_cache_does_not_keep_blocks_alive(vc):
    # the packed-weight cache holds a weak reference: a collected BlockParams
    # releases its device copy
    import gc
    import torch
    from paper_2501_08453_b200 import model as M
    blk = vc.BlockParams.init(vc.SeededRng(5).split(1000), 64)
    db = M.device_block(torch, blk, 4, "bf16")
    key = (id(blk), 4, "bf16")
    assert M._BLOCK_CACHE[key][1] is db
    assert M.device_block(torch, blk, 4, "bf16") is db  # unchanged weights: cached
    del blk
    gc.collect()
    assert key not in M._BLOCK_CACHE


# ---- 2B shapes (dh = 66), reduced frame counts so the fp64 oracle takes seconds ----

@pytest.mark.parametrize("F", [1, 2])
def test_2b_block_reduced_frames(vc, F):
    Lv, Lt, D, H = 1350, 256, 1584, 24
    blk, x, prompt = block_case(vc, f"2b_f{F}", F, Lv, Lt, D)
    text = vc.anchor_text(prompt, F)
    oblk = O.BlockParams(*[O.BranchParams(*br.arrays()) for br in blk.branches()])
    ref = O.parallel_block_forward(oblk, x, text, H)
    got32 = vc.parallel_block_forward(blk, x, text, H, dtype="fp32")
    assert normwise(got32, ref) <= FP32_TOL
    got16 = vc.parallel_block_forward(blk, x, text, H, dtype="bf16")
    assert rel_l2(got16, ref) <= BF16_TOL


def test_config5_shape_reduced_frames(vc):
    # temporal-dominant config 5 shape (D 3072, H 24, dh 128), F reduced 64 -> 4
    F, Lv, Lt, D, H = 4, 256, 256, 3072, 24
    blk, x, prompt = block_case(vc, "cfg5_f4", F, Lv, Lt, D)
    text = vc.anchor_text(prompt, F)
    oblk = O.BlockParams(*[O.BranchParams(*br.arrays()) for br in blk.branches()])
    ref = O.parallel_block_forward(oblk, x, text, H)
    assert rel_l2(vc.parallel_block_forward(blk, x, text, H, dtype="bf16"), ref) <= BF16_TOL
    assert normwise(vc.parallel_block_forward(blk, x, text, H, dtype="fp32"), ref) <= FP32_TOL


def test_config2_full_bf16_vs_fp32_transitive(vc):
    # Full config 2 (F=16): the fp64 oracle needs ~5 min / 24 GB, so parity is
    # transitive: bf16 vs the fp32 GPU path, which is oracle-checked above.
    import torch
    F, Lv, Lt, D, H = 16, 1350, 256, 1584, 24
    blk, x, prompt = block_case(vc, "cfg2", F, Lv, Lt, D)
    xt = torch.from_numpy(x.astype(np.float32)).cuda()
    text = vc.anchor_text(torch.from_numpy(prompt.astype(np.float32)).cuda(), F)
    y32 = vc.parallel_block_forward(blk, xt, text, H, dtype="fp32").double().cpu().numpy()
    y16 = vc.parallel_block_forward(blk, xt, text, H, dtype="bf16").double().cpu().numpy()
    assert np.isfinite(y16).all()
    assert rel_l2(y16, y32) <= BF16_TOL


def test_host_stream_matches_device_forward(vc):
    # serving path (vc_block_forward_host_batched): each batch equals the
    # single device-resident forward of the same input
    import torch
    from paper_2501_08453_b200.model import block_forward_host_stream
    F, Lv, Lt, D, H = 3, 64, 32, 256, 8
    blk, x, prompt = block_case(vc, "stream", F, Lv, Lt, D)
    xs = [torch.from_numpy((x * (i + 1)).astype(np.float32)).pin_memory() for i in range(5)]
    pt = torch.from_numpy(prompt.astype(np.float32)).pin_memory()
    for dt in ("fp32", "bf16"):
        outs = block_forward_host_stream(blk, xs, pt, H, dtype=dt)
        torch.cuda.synchronize()
        for i in range(5):
            ref = vc.parallel_block_forward(blk, x * (i + 1), vc.anchor_text(prompt, F), H, dtype=dt)
            assert np.array_equal(outs[i].double().numpy(), ref), (dt, i)
        # the serving handle (device-resident packed weights) gives the same bits
        from paper_2501_08453_b200.model import device_block
        outs2 = block_forward_host_stream(device_block(torch, blk, H, dt), xs, pt, H)
        torch.cuda.synchronize()
        for i in range(5):
            assert torch.equal(outs2[i], outs[i]), (dt, i)
        with pytest.raises(ValueError):
            block_forward_host_stream(device_block(torch, blk, H, dt), xs, pt, H + 1)


@pytest.mark.parametrize("F,Lv,D,H", [(16, 40, 1584, 24), (37, 9, 256, 2), (64, 8, 3072, 24), (160, 3, 1584, 24)])
def test_temporal_branch_long_clips(vc, F, Lv, D, H):
    # frame-axis attention over 16..160 frames (configs 2, 4, 5): tensor-core
    # (bf16) and smem / generic (fp32) kernels against the oracle
    r = vc.SeededRng(F * 1000 + D)
    p = vc.BranchParams.init(r.split(1), D)
    x = r.normal((F, Lv, D))
    ref = O.temporal_branch(O.BranchParams(*p.arrays()), x, H)
    assert normwise(vc.temporal_branch(p, x, H, dtype="fp32"), ref) <= FP32_TOL
    assert rel_l2(vc.temporal_branch(p, x, H, dtype="bf16"), ref) <= BF16_TOL


def test_block_random_shapes_sweep(vc):
    # seeded sweep over block geometries (frames, visual / text lengths incl.
    # zero text, dims, heads) against the oracle, both precisions; bf16 where
    # its layout constraints hold (dim % 8 == 0, head dim <= 128)
    rng = np.random.default_rng(2501_08453)
    for case in range(16):
        F = int(rng.integers(1, 5))
        Lv = int(rng.integers(1, 40))
        Lt = int(rng.choice([0, 1, 3, 16]))
        H = int(rng.choice([1, 2, 3, 4]))
        dh = int(rng.choice([4, 8, 16, 24, 32, 48, 66]))
        D = H * dh
        blk = vc.BlockParams.init(vc.SeededRng(1000 + case).split(1000), D)
        x = rng.standard_normal((F, Lv, D))
        prompt = rng.standard_normal((Lt, D))
        text = vc.anchor_text(prompt, F)
        oblk = O.BlockParams(*[O.BranchParams(*b.arrays()) for b in blk.branches()])
        ref = O.parallel_block_forward(oblk, x, O.anchor_text(prompt, F), H)
        got32 = vc.parallel_block_forward(blk, x, text, H, dtype="fp32")
        assert normwise(got32, ref) <= FP32_TOL, (case, F, Lv, Lt, D, H)
        if D % 8 == 0:
            got16 = vc.parallel_block_forward(blk, x, text, H, dtype="bf16")
            assert rel_l2(got16, ref) <= BF16_TOL, (case, F, Lv, Lt, D, H, rel_l2(got16, ref))


def test_vae_encode_and_fused_q_sample_vs_golden(vc):
    # the frame encoder + forward noising every rank runs on its round-robin
    # frames (executor.py:535-546): vc_vae_encode_frames vs the reference
    import torch

    from paper_2501_08453_b200.diffusion import make_linear_schedule
    from paper_2501_08453_b200.model import encode_frames_device
    sched = make_linear_schedule(100)
    for h, w, c in ((32, 32, 4), (37, 29, 4), (20, 50, 8)):
        frame = vc.SeededRng(900 + h).uniform((h, w, 3))
        spec = vc.PatchSpec(8, 2, c)
        lat = vc.toy_vae_encode(frame, spec)
        assert normwise(lat, G[f"vae_{h}x{w}_c{c}"]) <= 1e-6
        noise = vc.SeededRng(950 + h).normal(lat.shape)
        px = torch.from_numpy(frame[None].astype(np.float32)).cuda()
        nz = torch.from_numpy(noise[None].astype(np.float32)).cuda()
        got = encode_frames_device(torch, px, spec, sched, 37, nz)[0].double().cpu().numpy()
        assert normwise(got, G[f"qs37_{h}x{w}_c{c}"]) <= 1e-6
    with pytest.raises(ValueError, match="pixels"):
        vc.toy_vae_encode(np.zeros((8, 8, 4)))


def test_block_forward_captures_into_a_cuda_graph(vc):
    # the bf16 block forks its text K/V GEMM and temporal branch onto a side
    # stream and joins them back with events (vc_block_bf16.cu): the whole
    # forward must capture into one CUDA graph and replay to the same bits
    import torch

    from paper_2501_08453_b200.model import DeviceBlock, block_forward_device
    blk, x, prompt = block_case(vc, "blk_graph", 3, 40, 8, 264)  # dh 66: compact QKV, pad fills, side stream
    db = DeviceBlock(torch, blk, 4, "bf16")
    xt = torch.from_numpy(x.astype(np.float32)).cuda()
    pt = torch.from_numpy(prompt.astype(np.float32)).cuda()
    ref = torch.empty_like(xt)
    block_forward_device(torch, db, xt, pt, ref, False)  # warm: attributes, workspace
    out = torch.zeros_like(xt)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        block_forward_device(torch, db, xt, pt, out, False)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)

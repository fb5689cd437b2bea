"""GPU parity at the full BASELINE shapes, pinned to the fp64 oracle on
sampled rows (the full fp64 forward takes minutes to hours there).

For each shape the CUDA block runs over the WHOLE clip (every kernel at its
real grid: 1350-token frames with their 70-row tail tile, the 16 / 64 /
160-frame full sequence with its text keys deduplicated); the oracle
(`oracle.spsim_oracle.parallel_block_rows`) computes, in float64 and for just
the sampled query rows, everything those rows attend to (model.py:230-271).
Each branch is checked on its own (the other two branches zeroed, which
makes their contribution exactly 0) and summed as the block.

Rows are sampled from the first, second, middle and last frames and from
the positions next to the frame's text (l = 0, 1, 2 follow the text slots
in the checkerboard sequence, model.py:133-140), the attention tile edges,
and the last partial 128-row tile (rows 1280-1349 at Lv = 1350).

Tolerances (BASELINE.json north_star): bf16 relative L2 <= 2e-2 per branch
and per block over the sampled rows; fp32 normwise max|err| / max|ref| <= 1e-4.
"""
import numpy as np
import pytest

from oracle import spsim_oracle as O

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
FP32_TOL = 1e-4


def rel_l2(y, ref):
    return float(np.linalg.norm(y - ref) / np.linalg.norm(ref))


def normwise(y, ref):
    return float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


def sample_rows(F, Lv, n_frames=8, n_pos=32, seed=0):
    """>= 256 (frame, position) rows: cartesian product of sampled frames and
    positions, edge cases first."""
    rng = np.random.default_rng(seed)
    frames = [0, 1, F // 2, F - 1]
    rest = [f for f in range(F) if f not in frames]
    frames += list(rng.choice(rest, size=min(n_frames - len(frames), len(rest)), replace=False))
    tail0 = (Lv - 1) // 128 * 128  # first row of the last (partial) query tile
    pos = {0, 1, 2, 3, 127, 128, 255, 256, Lv - 1, Lv - 2, Lv - 3, tail0, tail0 + 1,
           (tail0 + Lv) // 2, max(tail0 - 1, 0)}
    pos = sorted(p for p in pos if 0 <= p < Lv)
    rest = [p for p in range(Lv) if p not in pos]
    pos += list(rng.choice(rest, size=max(n_pos - len(pos), 0), replace=False))
    fi = np.repeat(np.array(frames, dtype=np.int64), len(pos))
    li = np.tile(np.array(pos, dtype=np.int64), len(frames))
    return fi, li


def _branch_only(vc, blk, which, D):
    z = vc.BranchParams.zeros(D)
    parts = [z, z, z]
    parts[which] = blk.branches()[which]
    return vc.BlockParams(*parts)


def gpu_rows(torch, vc, blk, H, dtype, xt, pt, fi, li, branches=True):
    """Block output rows (and each branch's, other branches zeroed) of the
    CUDA forward over the whole clip."""
    from paper_2501_08453_b200.model import DeviceBlock, block_forward_device
    D = xt.shape[2]
    fidx = torch.from_numpy(fi).cuda()
    lidx = torch.from_numpy(li).cuda()
    out = torch.empty_like(xt)
    got = {}
    todo = [("block", blk)]
    if branches:
        todo += [(name, _branch_only(vc, blk, i, D)) for i, name in enumerate(("spatial", "temporal", "fullseq"))]
    for name, b in todo:
        db = DeviceBlock(torch, b, H, dtype)
        block_forward_device(torch, db, xt, pt, out, False)
        torch.cuda.synchronize()
        assert torch.isfinite(out).all().item(), name
        got[name] = out[fidx, lidx].double().cpu().numpy()
        del db
    return got


def make_case(vc, seed, F, Lv, Lt, D):
    blk = vc.BlockParams.init(vc.SeededRng(seed).split(1000), D)
    data = vc.SeededRng(seed).split(1 << 20)
    x = data.split(1).normal((F, Lv, D))
    prompt = data.split(2).normal((Lt, D))
    oblk = O.BlockParams(*[O.BranchParams(*b.arrays()) for b in blk.branches()])
    return blk, oblk, x, prompt


SHAPES = [
    # id, (F, Lv, Lt, D, H), fp32 path too
    ("config2_f16", (16, 1350, 256, 1584, 24), True),
    ("config5_f64", (64, 256, 256, 3072, 24), True),
    ("config4_f160", (160, 1350, 256, 1584, 24), False),
]


@pytest.mark.parametrize("case", SHAPES, ids=[s[0] for s in SHAPES])
def test_full_shape_block_vs_fp64_rows(torch, case):
    import paper_2501_08453_b200 as vc
    name, (F, Lv, Lt, D, H), fp32 = case
    blk, oblk, x, prompt = make_case(vc, sum(map(ord, name)), F, Lv, Lt, D)
    fi, li = sample_rows(F, Lv)
    assert fi.size >= 256
    ref = O.parallel_block_rows(oblk, x, O.anchor_text(prompt, F), H, fi, li)
    xt = torch.from_numpy(x.astype(np.float32)).cuda()
    pt = torch.from_numpy(prompt.astype(np.float32)).cuda()
    del x
    got = gpu_rows(torch, vc, blk, H, "bf16", xt, pt, fi, li)
    errs = {k: rel_l2(got[k], ref[k]) for k in got}
    print(name, "bf16 rel-L2", errs)
    for k, e in errs.items():
        assert e <= BF16_TOL, (k, e)
    # the rows next to the text and in the tail tile on their own
    for sel in (li <= 2, li >= (Lv - 1) // 128 * 128):
        assert rel_l2(got["block"][sel], ref["block"][sel]) <= BF16_TOL
    if fp32:
        got32 = gpu_rows(torch, vc, blk, H, "fp32", xt, pt, fi, li, branches=False)
        e32 = normwise(got32["block"], ref["block"])
        print(name, "fp32 normwise", e32)
        assert e32 <= FP32_TOL


def test_config3_model_depth2_vs_fp64_rows(torch):
    """Config 3 geometry (480p, 40 frames: 60x90 latents -> 30x45 patches, 256
    text tokens, D 1584, H 24) at depth 2: the embed over the whole clip
    (model.py:303-314, every row), each block's update on sampled rows given
    its input state (model.py:316-325 -- per-block north-star tolerance), and
    the unembed of the final state (model.py:327-333, every row); the public
    ToyDenoiser.forward equals the chained device pieces."""
    import paper_2501_08453_b200 as vc
    from paper_2501_08453_b200.model import DeviceBlock, block_forward_device
    from paper_2501_08453_b200.numerics import to_device_f32
    seed, F, h, w, Lt, D, H, depth, t = 2026, 40, 60, 90, 256, 1584, 24, 2, 37
    model = vc.ToyDenoiser.init(vc.SeededRng(seed), vc.PatchSpec(8, 2, 4), D, H, depth)
    om = O.ToyDenoiser(O.PatchSpec(8, 2, 4), D, H, model.w_in, model.w_out,
                       [O.BlockParams(*[O.BranchParams(*br.arrays()) for br in b.branches()]) for b in model.blocks])
    data = vc.SeededRng(seed).split(1 << 20)
    lat = data.split(1).normal((F, h, w, 4))
    prompt = data.split(2).normal((Lt, D))
    Lv = (h // 2) * (w // 2)
    lat_d = to_device_f32(torch, lat)
    pr_d = to_device_f32(torch, prompt)
    x = model._embed(torch, lat_d, 0, t)
    x0 = np.stack([om.embed_frame(lat[f], f, t) for f in range(F)])
    assert normwise(x.double().cpu().numpy(), x0) <= 1e-6
    fi, li = sample_rows(F, Lv, seed=3)
    fidx, lidx = torch.from_numpy(fi).cuda(), torch.from_numpy(li).cuda()
    text = O.anchor_text(prompt, F)
    for k, b in enumerate(model.blocks):
        x_in = x.double().cpu().numpy()
        db = DeviceBlock(torch, b, H, "bf16")
        x_next = torch.empty_like(x)
        block_forward_device(torch, db, x, pr_d, x_next, True)
        upd = (x_next[fidx, lidx].double() - x[fidx, lidx].double()).cpu().numpy()
        ref = O.parallel_block_rows(om.blocks[k], x_in, text, H, fi, li)["block"]
        e = rel_l2(upd, ref)
        print("config3 block", k, "bf16 rel-L2", e)
        assert e <= BF16_TOL, (k, e)
        x = x_next
    x2 = x.double().cpu().numpy()
    eps_ref = np.stack([O.unpatchify(x2[f] @ om.w_out, h, w, 4, 2) for f in range(F)])
    eps = model.forward(lat, t, prompt, dtype="bf16")
    assert normwise(eps, eps_ref) <= 1e-5

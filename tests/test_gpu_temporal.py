"""The temporal branch (model.py:238-244) against the fp64 oracle, through
the public block API with the spatial and full-sequence branches zeroed
(their contribution is then exactly 0), on both bf16 kernels: the tcgen05 +
TMA one (vc_attn_temporal_tc.cu; forced with the C-ABI switch
vc_set_temporal_impl) and the mma.sync one, both reading the position-major
q/k/v rows the QKV GEMM writes. Shapes cover the kernel's cases: npos = 128/F positions
per CTA with a partial last group (F = 16, 40, 5), one position in two
query tiles (F = 130, 160), head dims 64 / 66 (padded to 80, Q's padding
zeroed in shared memory) / 128, key counts that need zero padding rows
(F = 5: 125 keys in a 128-key tile; F = 40: 120)."""
import numpy as np
import pytest

from oracle import spsim_oracle as O

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2

SHAPES = [
    (16, 200, 8, 1584, 24),
    (40, 70, 8, 1584, 24),
    (160, 9, 8, 1584, 24),
    (130, 5, 8, 528, 8),
    (64, 20, 8, 3072, 24),
    (5, 77, 8, 512, 8),
    (64, 33, 8, 256, 4),
]


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


@pytest.mark.parametrize("impl", [2, 1], ids=["tcgen05", "mma_sync"])
@pytest.mark.parametrize("shape", SHAPES, ids=["x".join(map(str, s)) for s in SHAPES])
def test_temporal_branch_vs_oracle(torch, shape, impl):
    import paper_2501_08453_b200 as vc
    from paper_2501_08453_b200 import _lib
    lib = _lib.load()
    assert lib.vc_set_temporal_impl(impl) == 0
    from paper_2501_08453_b200.model import DeviceBlock, block_forward_device
    F, Lv, Lt, D, H = shape
    seed = F * 1000 + Lv
    full = vc.BlockParams.init(vc.SeededRng(seed).split(1000), D)
    z = vc.BranchParams.zeros(D)
    blk = vc.BlockParams(z, full.temporal, z)
    x = vc.SeededRng(seed).split(1).normal((F, Lv, D))
    prompt = vc.SeededRng(seed).split(2).normal((Lt, D))
    ref = O.temporal_branch(O.BranchParams(*full.temporal.arrays()), x, H)
    xt = torch.from_numpy(x.astype(np.float32)).cuda()
    pt = torch.from_numpy(prompt.astype(np.float32)).cuda()
    out = torch.empty_like(xt)
    block_forward_device(torch, DeviceBlock(torch, blk, H, "bf16"), xt, pt, out, False)
    got = out.double().cpu().numpy()
    assert np.isfinite(got).all()
    err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert err <= BF16_TOL, err
    # every position and frame is covered: per-(frame, position) rows match too
    rows = np.linalg.norm(got - ref, axis=2) / np.maximum(np.linalg.norm(ref, axis=2), 1e-30)
    assert float(rows.max()) <= 0.1, float(rows.max())
    assert lib.vc_set_temporal_impl(0) == 0

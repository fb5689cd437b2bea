"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `spsim` from /root/reference/pkg/src (read-only, no writes) and
stores the reference's own outputs in tests/golden/*.npz. The fixtures pin
the oracle (`oracle/spsim_oracle.py`) and, through it, the CUDA path.
Inputs are NOT stored (they are regenerated from seeds with SeededRng);
a checksum of every input stream is stored so a numpy whose Philox/normal
stream drifted is detected instead of silently compared.

Seeding convention (also used by tests and bench.py):
  model/block weights : SeededRng(seed) (ToyDenoiser.init) or
                        SeededRng(seed).split(1000) (BlockParams.init)
  inputs              : data = SeededRng(seed).split(1 << 20)
                        x / latents = data.split(1).normal(...)
                        prompt      = data.split(2).normal((Lt, D))
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from spsim import executor as rex  # noqa: E402
from spsim import model as rm  # noqa: E402
from spsim import numerics as rn  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
DATA_TAG = 1 << 20

# (name, F, Lv, Lt, D, H) block cases: config-1 block shape, ragged small
# shapes, dh not a power of two, and reduced-F variants of the 2B shape.
BLOCK_CASES = [
    ("blk_tiny", 4, 64, 32, 256, 4),
    ("blk_small", 3, 5, 2, 12, 4),
    ("blk_odd", 2, 7, 3, 18, 3),
    ("blk_dh66", 2, 24, 8, 132, 2),
]
MODEL_CASES = [
    # name, seed, F, latent h, w, Lt, D, H, depth, t
    ("cfg1", 2501, 4, 16, 16, 32, 256, 4, 2, 37),
    ("mdl_ragged", 7, 3, 5, 7, 3, 12, 6, 1, 11),
]


def block_inputs(seed, F, Lv, Lt, D):
    data = rn.SeededRng(seed).split(DATA_TAG)
    x = data.split(1).normal((F, Lv, D))
    prompt = data.split(2).normal((Lt, D))
    return x, prompt


def main():
    fixtures = {}
    # --- RNG stream pins -------------------------------------------------
    r = rn.SeededRng(123456789)
    fixtures["rng_normal_head"] = r.normal(64)
    fixtures["rng_split_head"] = rn.SeededRng(42).split(1000).split(101).normal(16)

    # --- attention / softmax known answers -------------------------------
    g = rn.SeededRng(21)
    q, k, v = g.normal((10, 8)), g.normal((13, 8)), g.normal((13, 8))
    fixtures["attn_q"], fixtures["attn_k"], fixtures["attn_v"] = q, k, v
    for h in (1, 2, 4):
        fixtures[f"attn_out_h{h}"] = rn.attention(q, k, v, h)
    fixtures["softmax_pair"] = rn.softmax_rows(np.array([[0.0, np.log(3.0)]]))

    # --- block forwards --------------------------------------------------
    for name, F, Lv, Lt, D, H in BLOCK_CASES:
        seed = sum(map(ord, name))
        blk = rm.BlockParams.init(rn.SeededRng(seed).split(1000), D)
        x, prompt = block_inputs(seed, F, Lv, Lt, D)
        text = rm.anchor_text(prompt, F)
        fixtures[f"{name}_seed"] = np.array(seed)
        fixtures[f"{name}_xsum"] = np.array([x.sum(), prompt.sum(), blk.fullseq.wo.sum()])
        fixtures[f"{name}_sp"] = rm.spatial_branch(blk.spatial, x, H)
        fixtures[f"{name}_tm"] = rm.temporal_branch(blk.temporal, x, H)
        fixtures[f"{name}_fs"] = rm.full_sequence_attention(blk.fullseq, text, x, H)
        fixtures[f"{name}_out"] = rm.parallel_block_forward(blk, x, text, H)
        print(name, "done", flush=True)

    # --- model forwards --------------------------------------------------
    for name, seed, F, h, w, Lt, D, H, depth, t in MODEL_CASES:
        spec = rm.PatchSpec(8, 2, 4)
        model = rm.ToyDenoiser.init(rn.SeededRng(seed), spec, D, H, depth)
        data = rn.SeededRng(seed).split(DATA_TAG)
        lat = data.split(1).normal((F, h, w, 4))
        prompt = data.split(2).normal((Lt, D))
        fixtures[f"{name}_xsum"] = np.array([lat.sum(), prompt.sum(), model.w_out.sum()])
        fixtures[f"{name}_embed0"] = model.embed_frame(lat[0], 0, t)
        fixtures[f"{name}_states"] = model.head_states(lat, t, prompt)
        fixtures[f"{name}_out"] = model.forward(lat, t, prompt)
        print(name, "done", flush=True)

    # --- one full sampling step on the config-1 model (diffusion.py:95-116) -
    from spsim.diffusion import make_linear_schedule, reverse_step
    sched = make_linear_schedule(100)
    spec = rm.PatchSpec(8, 2, 4)
    model = rm.ToyDenoiser.init(rn.SeededRng(2501), spec, 256, 4, 2)
    data = rn.SeededRng(2501).split(DATA_TAG)
    lat = data.split(1).normal((4, 16, 16, 4))
    prompt = data.split(2).normal((32, 256))
    z = data.split(3).normal((4, 16, 16, 4))
    for t in (37, 1):
        eps = model.forward(lat, t, prompt)
        fixtures[f"rev_t{t}"] = reverse_step(sched, lat, t, eps, z)
    fixtures["sched100_betas"] = sched.betas

    # --- integer shard maps (exact) --------------------------------------
    rows = []
    for n in (1, 2, 3, 5, 7, 32, 36, 64, 256, 1350, 1351):
        for p in (1, 2, 3, 4, 5, 6, 7, 8, 16):
            rows.append((n, p, rex.contiguous_bounds(n, p)))
    fixtures["cb_np"] = np.array([(n, p) for n, p, _ in rows])
    fixtures["cb_flat"] = np.concatenate([np.array(b) for _, _, b in rows])
    pd_rows = []
    for lt, lv in ((32, 64), (256, 1350), (3, 4), (6, 36), (1, 7)):
        for p in (1, 2, 3, 4, 6, 8):
            for plc in ("separate", "fused"):
                tc, vc = rex.placement_division(lt, lv, p, plc)
                pd_rows.append([lt, lv, p, int(plc == "fused")] + list(tc) + list(vc))
    fixtures["pd_rows"] = np.array([r + [-1] * (4 + 16 - len(r)) for r in pd_rows])
    fixtures["rr_10_4"] = np.array([len(d) for d in rex.round_robin_frames(10, 4)])

    # --- sharded == single device, reference executor (acceptance crit. 1)
    from spsim.cluster import ClusterSpec
    from spsim.diffusion import make_linear_schedule
    spec = rm.PatchSpec(8, 2, 4)
    model = rm.ToyDenoiser.init(rn.SeededRng(77), spec, dim=12, heads=6, depth=1)
    sched = make_linear_schedule(100)
    batch = rex.make_batch(20240701, 3, 32, 32, 3, 12)
    ref = rex.reference_iteration(model, sched, batch)
    fixtures["sp_ref_pred"] = ref.predicted_noise
    for p in (2, 3):
        res = rex.run_sp_iteration(model, sched, batch,
                                   rex.ShardingPlan(p, "spatial", "head_parallel", "separate"),
                                   ClusterSpec(nodes=1, devices_per_node=8))
        fixtures[f"sp_p{p}_pred"] = res.predicted_noise
        fixtures[f"sp_p{p}_comm"] = np.array([e.bytes_per_device for e in res.log.events])

    # --- toy VAE encode (model.py:381-403) and q_sample (diffusion.py:77-84):
    # ragged frame sizes (zero padding), 4 and 8 latent channels
    from spsim.diffusion import q_sample
    for h, w, c in ((32, 32, 4), (37, 29, 4), (20, 50, 8)):
        frame = rn.SeededRng(900 + h).uniform((h, w, 3))
        lat = rm.toy_vae_encode(frame, rm.PatchSpec(8, 2, c))
        fixtures[f"vae_{h}x{w}_c{c}"] = lat
        noise = rn.SeededRng(950 + h).normal(lat.shape)
        fixtures[f"qs37_{h}x{w}_c{c}"] = q_sample(sched, lat, 37, noise)

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **fixtures)
    print("wrote", os.path.join(OUT, "golden.npz"))


if __name__ == "__main__":
    main()

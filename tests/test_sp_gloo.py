"""Multi-process sequence parallelism on CPU: world_size 2 and 3 over gloo,
the product's driver (sp.run_stages) and exchange (sp.TorchExchange, i.e.
torch.distributed.all_to_all_single with the product's per-peer counts),
numpy stand-ins for the CUDA stages. The gathered sharded result must equal
the single-device oracle block (reference acceptance criterion 1:
tests/test_acceptance.py:51-72, sharded == reference)."""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SHAPE = dict(F=3, Lv=7, Lt=3, D=24, H=6)


def _case(sh=SHAPE):
    from oracle import spsim_oracle as O
    F, Lv, Lt, D = sh["F"], sh["Lv"], sh["Lt"], sh["D"]
    blk = O.BlockParams.init(O.SeededRng(77).split(1000), D)
    data = O.SeededRng(77).split(1 << 20)
    return blk, data.split(1).normal((F, Lv, D)), data.split(2).normal((Lt, D))


def _worker(rank, world, port, outdir, add_residual, mode="head_parallel", shape=None):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from paper_2501_08453_b200 import sp
    from sp_numpy_stages import NumpyGatherStages, NumpyStages
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shape or SHAPE
        blk, x, prompt = _case(sh)
        if mode == "gather":
            st = NumpyGatherStages(blk, sh["F"], sh["Lv"], sh["Lt"], sh["D"], sh["H"], world, rank)
            run = sp.run_gather_stages
        else:
            st = NumpyStages(blk, sh["F"], sh["Lv"], sh["Lt"], sh["D"], sh["H"], world, rank)
            run = sp.run_stages
        lo, hi = st.vb[rank], st.vb[rank + 1]
        xl = torch.from_numpy(np.ascontiguousarray(x[:, lo:hi]))
        out = torch.empty_like(xl)
        run(st, xl, torch.from_numpy(prompt), out, sp.TorchExchange(), add_residual)
        np.save(os.path.join(outdir, f"out{rank}.npy"), out.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,add_residual", [(2, False), (3, True)])
def test_sp_gloo_equals_single_device(world, add_residual):
    from oracle import spsim_oracle as O
    blk, x, prompt = _case()
    ref = O.parallel_block_forward(blk, x, O.anchor_text(prompt, SHAPE["F"]), SHAPE["H"])
    if add_residual:
        ref = ref + x
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, add_residual), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(d, f"out{r}.npy")) for r in range(world)], axis=1)
    np.testing.assert_allclose(got, ref, atol=1e-10, rtol=0)


# gather mode (executor.py:416-459): P need not divide H (4 heads on 3 ranks)
GATHER_SHAPE = dict(F=3, Lv=7, Lt=3, D=16, H=4)


@pytest.mark.parametrize("world,add_residual", [(2, True), (3, False)])
def test_sp_gather_gloo_equals_single_device(world, add_residual):
    from oracle import spsim_oracle as O
    sh = GATHER_SHAPE
    blk, x, prompt = _case(sh)
    ref = O.parallel_block_forward(blk, x, O.anchor_text(prompt, sh["F"]), sh["H"])
    if add_residual:
        ref = ref + x
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, add_residual, "gather", sh), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(d, f"out{r}.npy")) for r in range(world)], axis=1)
    np.testing.assert_allclose(got, ref, atol=1e-10, rtol=0)


def _log_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import json

    import torch.distributed as dist

    from paper_2501_08453_b200 import sp
    from sp_numpy_stages import NumpyStages
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = SHAPE
        blk, x, prompt = _case(sh)
        st = NumpyStages(blk, sh["F"], sh["Lv"], sh["Lt"], sh["D"], sh["H"], world, rank)
        lo, hi = st.vb[rank], st.vb[rank + 1]
        xl = torch.from_numpy(np.ascontiguousarray(x[:, lo:hi]))
        log = sp.CommLog()
        ex = sp.LoggedExchange(sp.TorchExchange(), log, world, bpe=8)  # the stand-in exchanges fp64
        sp.run_stages(st, xl, torch.from_numpy(prompt), torch.empty_like(xl), ex, stage_prefix="block0")
        with open(os.path.join(outdir, f"log{rank}.json"), "w") as f:
            json.dump([[*e.key(), e.payload_bytes] for e in log.events], f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_logged_collectives_match_reference_comm_plan(world):
    # the CommLog of the collectives the product's driver really issues
    # (executor.py:111-141 fields) against the reference's schedule
    # (executor.py:721-773, oracle.comm_plan, pinned to the reference's log):
    # same stages, collectives, group and placement in the same order; the
    # payload bytes (largest rank, as the reference logs) equal, except the
    # full-sequence a2a #1, which does not ship the text rows (every rank
    # projects them from its own prompt copy); no "reshard" (each rank embeds
    # its own rows) -- and the "gather" is sp_model_forward's, not run_stages'
    import json

    from oracle import spsim_oracle as O
    sh = SHAPE
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_log_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        logs = [json.load(open(os.path.join(d, f"log{r}.json"))) for r in range(world)]
    ref = O.comm_plan(sh["F"], sh["Lt"], sh["Lv"], sh["D"], sh["H"], 1, world)
    ref_block = [r for r in ref if r[0].startswith("block0")]
    # issue order differs by design (both branches' a2a #1 go out before
    # either attention, to overlap them): compare each stage's own sequence
    order = {"block0.spatial": 0, "block0.fullseq": 1}
    logs = [sorted(log, key=lambda e: order[e[0]]) for log in logs]  # stable: per-stage order kept
    assert all([tuple(e[:4]) for e in log] == [tuple(r[:4]) for r in ref_block] for log in logs)
    payload = [max(log[i][5] for log in logs) for i in range(len(ref_block))]
    tb = O.contiguous_bounds(sh["Lt"], world)
    text_rows = sh["F"] * max(tb[r + 1] - tb[r] for r in range(world))
    expect = [r[4] for r in ref_block]
    expect[2] -= 3 * text_rows * sh["D"] * 8  # full-sequence a2a #1: no text rows on the wire
    assert payload == expect

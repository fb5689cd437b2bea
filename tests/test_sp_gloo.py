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

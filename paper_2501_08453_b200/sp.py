"""Sequence-parallel block forward over one 8xB200 box (the paper's
memory-efficient hybrid-parallel scheme, spatial shard axis).

Reference: run_sp_iteration stage 3 (executor.py:561-626) with
_branch_head_parallel (executor.py:332-413): rank r holds visual rows
[vb[r], vb[r+1]) of every frame; the spatial and full-sequence branches
exchange q/k/v by head group (all-to-all #1), attend over full sequences for
H/P heads, and send the output columns back to the row owners (all-to-all
#2); the temporal branch is rank-local.

The three rank-local stages are CUDA (vc_sp_stage1/2/3 in the C ABI); the
two all-to-alls are NCCL `all_to_all_single` calls over NVLink/NVSwitch
issued here through torch.distributed (one process per GPU). An
`Exchange` object abstracts the collective so the same driver also runs
(a) a gloo world on CPU in the tests (with numpy stand-ins for the stages)
and (b) P virtual ranks in one process on one GPU for the parity test.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib


# ---------------------------------------------------------------------------
# Integer shard maps (exact restatements; executor.py:187-245)
# ---------------------------------------------------------------------------

def contiguous_bounds(n: int, p: int) -> list:
    """executor.py:187-191: p+1 split points, bounds[i] = i*n//p."""
    if p < 1:
        raise ValueError(f"cannot split into {p} parts")
    return [i * n // p for i in range(p + 1)]


def placement_division(text_len: int, visual_len: int, p: int, placement: str = "separate"):
    """executor.py:216-229 (the 'separate' placement the paper uses; 'fused'
    is the ablation baseline and is not run on the GPU path)."""
    if placement == "separate":
        tb, vb = contiguous_bounds(text_len, p), contiguous_bounds(visual_len, p)
        return [tb[i + 1] - tb[i] for i in range(p)], [vb[i + 1] - vb[i] for i in range(p)]
    if placement == "fused":
        b = contiguous_bounds(text_len + visual_len, p)
        out = []
        for lo, hi in zip(b[:-1], b[1:]):
            t = max(0, min(text_len, hi) - min(text_len, lo))
            out.append((t, hi - lo - t))
        return [t for t, _ in out], [v for _, v in out]
    raise ValueError(f"unknown text placement {placement!r}")


def prefix_bounds(counts) -> list:
    """executor.py:241-245."""
    out = [0]
    for c in counts:
        out.append(out[-1] + c)
    return out


def head_group_columns(dim: int, heads: int, p: int, g: int):
    """Columns of head group g: [g*D/P, (g+1)*D/P) = heads [g*H/P, (g+1)*H/P)
    (executor.py:336-337, :372-373)."""
    if heads % p:
        raise ValueError(f"head-parallel attention needs sp_size to divide {heads} heads, got {p}")
    w = dim // p
    return g * w, (g + 1) * w


def check_plan(frames, visual_len, heads, p):
    """executor.py:517-529 validity."""
    if p > visual_len:
        raise ValueError(f"cannot spread {visual_len} visual tokens per frame over {p} devices")
    if p > 1 and heads % p != 0:
        raise ValueError(f"head-parallel attention needs sp_size to divide {heads} heads, got {p}")


def exchange_counts(frames, visual_len, heads, dim, p, rank, padded=True):
    """Per-peer element counts of the two all-to-alls (bf16 elements), from
    the C ABI (vc_sp_exchange_elems) so the layout rule lives in one place:
    send1/recv1 carry q,k,v of 2 branches for H/P heads (head dim padded to
    DP); send2/recv2 carry 2 branches' attention outputs (H/P * dh, or H/P
    DP-wide head slots when dh is 66). padded=False gives the same exchanges
    without the layout padding (the reference's payload).
    The buffers are branch-major (vc_sp.cu): each branch is one half, split by
    peer with half these counts (branch_counts)."""
    lib = _lib.load()
    plan = _lib.SpPlan(_lib.shape(frames, visual_len, 0, dim, heads, "bf16"), p, rank)
    base = 0 if padded else 4
    out = {}
    for i, k in enumerate(("send1", "recv1", "send2", "recv2")):
        out[k] = [int(lib.vc_sp_exchange_elems(C.byref(plan), base + i, r)) for r in range(p)]
        if min(out[k]) < 0:
            raise ValueError(lib.vc_last_error().decode())
    return out


def branch_counts(counts):
    """Per-peer counts of ONE branch's exchange (half of every peer's block)."""
    return {k: [c // 2 for c in v] for k, v in counts.items()}


def head_pad(dh: int) -> int:
    return 64 if dh <= 64 else 80 if dh <= 80 else 128 if dh <= 128 else 0


# ---------------------------------------------------------------------------
# Collectives
# ---------------------------------------------------------------------------

class TorchExchange:
    """all_to_all_single over a torch.distributed group (NCCL on GPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def all_to_all(self, recv, send, recv_counts, send_counts, async_op=False):
        """Returns a handle with .wait() (the current stream waits for the
        collective; NCCL runs it on its own stream) when async_op. Nothing
        to move (one rank: the own block never enters the buffers) is no
        collective at all."""
        if len(send_counts) == 1 and not send_counts[0] and not recv_counts[0]:
            return _Done() if async_op else None
        return self.dist.all_to_all_single(recv, send, recv_counts, send_counts, group=self.group,
                                           async_op=async_op)

    def all_gather(self, gather, rank):
        """In place: gather is [P * slot]; this rank's slot is already filled."""
        n = gather.numel() // self.dist.get_world_size(self.group)
        self.dist.all_gather_into_tensor(gather, gather[rank * n:(rank + 1) * n], group=self.group)


class _Done:
    def wait(self):
        return None


@dataclass(frozen=True)
class CommEvent:
    """One collective this rank issued (executor.py:91-108's CommEvent fields;
    bytes_per_device is what this rank hands to the collective as laid out
    (its own block excluded: it never leaves the rank); payload_bytes the
    same exchange in the reference's payload terms: no layout padding, own
    block included, as the reference's executor logs it)."""
    stage: str
    collective: str
    group_size: int
    placement: str
    bytes_per_device: float
    payload_bytes: float = 0.0

    def key(self) -> tuple:
        return (self.stage, self.collective, self.group_size, self.placement, self.bytes_per_device)


@dataclass
class CommLog:
    """Ordered record of the collectives one forward issued (executor.py:111-141)."""
    events: list = field(default_factory=list)

    def record(self, stage, collective, group_size, placement, bytes_per_device, payload_bytes=0.0):
        self.events.append(CommEvent(stage, collective, int(group_size), placement, float(bytes_per_device),
                                     float(payload_bytes)))

    def rows(self) -> list:
        return [e.key() for e in self.events]


class LoggedExchange:
    """Wraps an exchange (TorchExchange: NCCL on the GPU box, gloo in the CPU
    tests) and records every collective run_stages / sp_model_forward issue
    into a CommLog, with the bytes actually handed to the collective."""

    def __init__(self, inner, log: CommLog, group_size: int, bpe: int = 2, placement: str = "intra"):
        self.inner, self.log, self.P, self.bpe, self.placement = inner, log, group_size, bpe, placement
        self.stage = "?"
        self.payload = None  # reference-payload element count of the next exchange (set by the driver)

    def all_to_all(self, recv, send, recv_counts, send_counts, async_op=False):
        self.log.record(self.stage, "alltoall", self.P, self.placement, sum(send_counts) * self.bpe,
                        (self.payload if self.payload is not None else sum(send_counts)) * self.bpe)
        self.payload = None
        return self.inner.all_to_all(recv, send, recv_counts, send_counts, async_op=async_op)

    def all_gather(self, gather, rank):
        n = gather.numel() // self.P
        self.log.record(self.stage, "allgather", self.P, self.placement, n * self.bpe, n * self.bpe)
        return self.inner.all_gather(gather, rank)


# ---------------------------------------------------------------------------
# The rank-local CUDA stages
# ---------------------------------------------------------------------------

class SPBlock:
    """One rank's share of a sequence-parallel block forward (bf16)."""

    def launches_per_forward(self) -> int:
        """Kernels this rank launches per forward (vc_sp.cu; NCCL's own not counted):
        stage 1 LN + QKV GEMM + temporal, stage 2 per branch an unpack of the
        peers' rows (P > 1) + text K/V GEMMs (2) + spatial + full-sequence
        attention, stage 3 unpack of the peers' groups (P > 1) + O GEMM."""
        mr = self.F * (self.vb[self.rank + 1] - self.vb[self.rank])
        peers = self.P > 1
        return ((3 if mr > 0 else 1) + (2 if peers else 0) + (2 if self.Lt > 0 else 0) + 2
                + ((2 if peers else 1) if mr > 0 else 0))

    def __init__(self, torch, device_block, frames, visual_len, text_len, nranks, rank):
        if device_block.dtype != "bf16":
            raise ValueError("sequence parallelism runs the bf16 path")
        self.torch = torch
        self.db = device_block
        D, H = device_block.dim, device_block.heads
        check_plan(frames, visual_len, H, nranks)
        self.plan = _lib.SpPlan(_lib.shape(frames, visual_len, text_len, D, H, "bf16"), nranks, rank)
        lib = _lib.load()
        _lib.check(lib.vc_sp_check(C.byref(self.plan)), "sp plan")
        self.F, self.Lv, self.Lt, self.D, self.H, self.P, self.rank = frames, visual_len, text_len, D, H, nranks, rank
        vb = (C.c_int32 * (nranks + 1))()
        _lib.check(lib.vc_sp_bounds(C.byref(self.plan), vb))
        self.vb = list(vb)
        self.counts = {k: [int(lib.vc_sp_exchange_elems(C.byref(self.plan), i, r)) for r in range(nranks)]
                       for i, k in enumerate(("send1", "recv1", "send2", "recv2"))}
        self.payload_counts = {k: [int(lib.vc_sp_exchange_elems(C.byref(self.plan), 4 + i, r)) for r in range(nranks)]
                               for i, k in enumerate(("send1", "recv1", "send2", "recv2"))}
        dev = "cuda"
        bf = torch.bfloat16
        self.send1 = torch.empty(sum(self.counts["send1"]), dtype=bf, device=dev)
        self.recv1 = torch.empty(sum(self.counts["recv1"]), dtype=bf, device=dev)
        self.send2 = torch.empty(sum(self.counts["send2"]), dtype=bf, device=dev)
        self.recv2 = torch.empty(sum(self.counts["recv2"]), dtype=bf, device=dev)
        self.ws_bytes = int(lib.vc_sp_workspace_bytes(C.byref(self.plan)))
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=dev)

    @property
    def local_rows(self):
        return self.vb[self.rank], self.vb[self.rank + 1]

    def stage1(self, x_local, prompt, part=2):
        """part 0: LN + QKV GEMM (fills send1), 1: temporal branch, 2: both."""
        lib = _lib.load()
        _lib.check(lib.vc_sp_stage1_part(C.byref(self.plan), _lib.ptr(self.db.packed), _lib.ptr(x_local),
                                         _lib.ptr(prompt) if self.Lt else C.c_void_p(0), _lib.ptr(self.send1),
                                         int(part), _lib.ptr(self.ws), self.ws_bytes,
                                         _lib.stream_ptr(self.torch)), "sp stage1")

    def stage2(self, branch=None):
        """Both branches, or one (0 spatial / 1 full sequence)."""
        lib = _lib.load()
        if branch is None:
            _lib.check(lib.vc_sp_stage2(C.byref(self.plan), _lib.ptr(self.db.packed), _lib.ptr(self.recv1),
                                        _lib.ptr(self.send2), _lib.ptr(self.ws), self.ws_bytes,
                                        _lib.stream_ptr(self.torch)), "sp stage2")
        else:
            _lib.check(lib.vc_sp_stage2_branch(C.byref(self.plan), _lib.ptr(self.db.packed), _lib.ptr(self.recv1),
                                               _lib.ptr(self.send2), int(branch), _lib.ptr(self.ws), self.ws_bytes,
                                               _lib.stream_ptr(self.torch)), "sp stage2")

    def stage3(self, x_local, out_local, add_residual=False):
        lib = _lib.load()
        _lib.check(lib.vc_sp_stage3(C.byref(self.plan), _lib.ptr(self.db.packed), _lib.ptr(self.recv2),
                                    _lib.ptr(x_local), _lib.ptr(out_local), 1 if add_residual else 0,
                                    _lib.ptr(self.ws), self.ws_bytes, _lib.stream_ptr(self.torch)), "sp stage3")

    def forward(self, x_local, prompt, out_local, exchange, add_residual=False, stage_prefix="block0"):
        """x_local [F, vc_r, D] fp32 -> out_local [F, vc_r, D] fp32 (block
        output of the local rows, + x_local if add_residual)."""
        return run_stages(self, x_local, prompt, out_local, exchange, add_residual, stage_prefix)


def _half(buf, b):
    n = buf.numel() // 2
    return buf[b * n:(b + 1) * n]


def run_stages(stages, x_local, prompt, out_local, exchange, add_residual=False, stage_prefix="block0"):
    """The rank-local schedule with the exchange split by branch (the buffers
    are branch-major) so it overlaps compute:

      stage1 part 0 (LN + QKV GEMM into send1)
        -> a2a#1 spatial, a2a#1 full-seq (async, NCCL stream)
      stage1 part 1 (the rank-local temporal branch, under a2a#1)
      wait spatial   -> stage2 spatial  -> a2a#2 spatial (async)
      wait full-seq  -> stage2 full-seq -> a2a#2 full-seq (async)
      wait both      -> stage3

    so the q/k/v travel while the temporal branch runs, the full-sequence
    q/k/v while the spatial attention runs, and the spatial outputs while the
    full-sequence attention runs. `stages` provides stage1/2/3, the four
    exchange buffers and per-peer counts (SPBlock on the GPU; a numpy
    stand-in in the CPU gloo test). With a LoggedExchange every collective is
    recorded under f"{stage_prefix}.spatial" / ".fullseq" (executor.py:571-626)."""
    bc = branch_counts(stages.counts)
    ref = getattr(stages, "payload_counts", None)
    ref = branch_counts(ref) if ref else None
    stages.stage1(x_local, prompt, part=0)
    h1 = []
    for b, name in ((0, "spatial"), (1, "fullseq")):
        if isinstance(exchange, LoggedExchange):
            exchange.stage = f"{stage_prefix}.{name}"
            exchange.payload = sum(ref["send1"]) if ref else None
        h1.append(exchange.all_to_all(_half(stages.recv1, b), _half(stages.send1, b), bc["recv1"], bc["send1"],
                                      async_op=True))
    stages.stage1(x_local, prompt, part=1)
    h2 = []
    for b, name in ((0, "spatial"), (1, "fullseq")):
        h1[b].wait()
        stages.stage2(b)
        if isinstance(exchange, LoggedExchange):
            exchange.stage = f"{stage_prefix}.{name}"
            exchange.payload = sum(ref["send2"]) if ref else None
        h2.append(exchange.all_to_all(_half(stages.recv2, b), _half(stages.send2, b), bc["recv2"], bc["send2"],
                                      async_op=True))
    for h in h2:
        h.wait()
    stages.stage3(x_local, out_local, add_residual)
    return out_local


class SPGatherBlock:
    """One rank's share of a GATHER-mode sequence-parallel block forward
    (_branch_gather, executor.py:416-459): all-gather the spatial and
    full-sequence K,V of all heads, attend for the own rows. No head
    divisibility requirement (P need not divide H); about 4x the exchange
    volume of the head-parallel mode, which stays the default."""

    def __init__(self, torch, device_block, frames, visual_len, text_len, nranks, rank):
        if device_block.dtype != "bf16":
            raise ValueError("sequence parallelism runs the bf16 path")
        self.torch = torch
        self.db = device_block
        D, H = device_block.dim, device_block.heads
        if nranks > visual_len:
            raise ValueError(f"cannot spread {visual_len} visual tokens per frame over {nranks} devices")
        self.plan = _lib.SpPlan(_lib.shape(frames, visual_len, text_len, D, H, "bf16"), nranks, rank)
        lib = _lib.load()
        _lib.check(lib.vc_spg_check(C.byref(self.plan)), "sp plan")
        self.F, self.Lv, self.Lt, self.D, self.H, self.P, self.rank = frames, visual_len, text_len, D, H, nranks, rank
        self.vb = contiguous_bounds(visual_len, nranks)
        self.slot = int(lib.vc_spg_slot_elems(C.byref(self.plan)))
        self.gather = torch.empty(nranks * self.slot, dtype=torch.bfloat16, device="cuda")
        self.ws_bytes = int(lib.vc_spg_workspace_bytes(C.byref(self.plan)))
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device="cuda")

    @property
    def local_rows(self):
        return self.vb[self.rank], self.vb[self.rank + 1]

    def launches_per_forward(self) -> int:
        """stage 1 LN + QKV GEMM + temporal + text K/V GEMM, stage 2 two unpack
        kernels + spatial + full-sequence attention + O GEMM (NCCL not counted)."""
        mr = self.F * (self.vb[self.rank + 1] - self.vb[self.rank])
        return 1 + (2 if mr > 0 else 0) + (1 if self.Lt > 0 else 0) + 2 + (3 if mr > 0 else 0)

    def stage1(self, x_local, prompt):
        lib = _lib.load()
        _lib.check(lib.vc_spg_stage1(C.byref(self.plan), _lib.ptr(self.db.packed), _lib.ptr(x_local),
                                     _lib.ptr(prompt) if self.Lt else C.c_void_p(0), _lib.ptr(self.gather),
                                     _lib.ptr(self.ws), self.ws_bytes, _lib.stream_ptr(self.torch)), "spg stage1")

    def stage2(self, x_local, out_local, add_residual=False):
        lib = _lib.load()
        _lib.check(lib.vc_spg_stage2(C.byref(self.plan), _lib.ptr(self.db.packed), _lib.ptr(self.gather),
                                     _lib.ptr(x_local), _lib.ptr(out_local), 1 if add_residual else 0,
                                     _lib.ptr(self.ws), self.ws_bytes, _lib.stream_ptr(self.torch)), "spg stage2")

    def forward(self, x_local, prompt, out_local, exchange, add_residual=False):
        return run_gather_stages(self, x_local, prompt, out_local, exchange, add_residual)


def run_gather_stages(stages, x_local, prompt, out_local, exchange, add_residual=False):
    """Gather-mode rank-local schedule: stage1 (this rank's K,V slot) ->
    in-place all-gather of the slots -> stage2 (SPGatherBlock on the GPU; a
    numpy stand-in in the CPU gloo test)."""
    stages.stage1(x_local, prompt)
    exchange.all_gather(stages.gather, stages.rank)
    stages.stage2(x_local, out_local, add_residual)
    return out_local


def emulate_sp_gather_forward(torch, device_block, x, prompt, nranks, add_residual=False):
    """Gather-mode SP block forward over P virtual ranks on one GPU (the
    all-gather becomes slot copies; ranks never wait on one another)."""
    F, Lv, D = x.shape
    Lt = prompt.shape[0] if prompt is not None else 0
    blocks = [SPGatherBlock(torch, device_block, F, Lv, Lt, nranks, r) for r in range(nranks)]
    vb = blocks[0].vb
    xs = [x[:, vb[r]:vb[r + 1]].contiguous() for r in range(nranks)]
    outs = [torch.empty_like(t) for t in xs]
    for r, b in enumerate(blocks):
        b.stage1(xs[r], prompt)
    n = blocks[0].slot
    for g in range(nranks):  # every rank receives every slot
        for r in range(nranks):
            if r != g:
                blocks[g].gather[r * n:(r + 1) * n].copy_(blocks[r].gather[r * n:(r + 1) * n])
    for r, b in enumerate(blocks):
        b.stage2(xs[r], outs[r], add_residual)
    return torch.cat(outs, dim=1)


class EmulatedRanks:
    """P virtual ranks in one process on one GPU: stage k of every rank, then
    the all-to-all as buffer copies with the product's per-peer counts. Used by
    the parity tests (a real multi-GPU run uses SPBlock.forward with
    TorchExchange; ranks here never wait on one another, so this is safe on
    one device)."""

    def __init__(self, torch, device_block, frames, visual_len, text_len, nranks):
        self.torch = torch
        self.P = nranks
        self.blocks = [SPBlock(torch, device_block, frames, visual_len, text_len, nranks, r)
                       for r in range(nranks)]
        self.vb = self.blocks[0].vb

    def _exchange(self, send_name, recv_name):
        # branch-major buffers: one all-to-all per branch half
        for br in (0, 1):
            for g in range(self.P):
                pieces = []
                for r in range(self.P):
                    b = self.blocks[r]
                    cnt = [c // 2 for c in b.counts[send_name]]
                    off = sum(cnt[:g])
                    pieces.append(_half(getattr(b, send_name), br)[off:off + cnt[g]])
                self.torch.cat(pieces, out=_half(getattr(self.blocks[g], recv_name), br))

    def block_forward(self, xs, prompt, outs, add_residual=False, device_block=None):
        """xs / outs: per-rank [F, vc_r, D] fp32 (outs may alias xs)."""
        for b in self.blocks:
            if device_block is not None:
                b.db = device_block
        for r, b in enumerate(self.blocks):
            b.stage1(xs[r], prompt)
        self._exchange("send1", "recv1")
        for b in self.blocks:
            b.stage2()
        self._exchange("send2", "recv2")
        for r, b in enumerate(self.blocks):
            b.stage3(xs[r], outs[r], add_residual)
        return outs

    def split(self, x):
        return [x[:, self.vb[r]:self.vb[r + 1]].contiguous() for r in range(self.P)]


def emulate_sp_forward(torch, device_block, x, prompt, nranks, add_residual=False):
    """One SP block forward over P virtual ranks; returns the gathered [F, Lv, D]."""
    F, Lv, D = x.shape
    Lt = prompt.shape[0] if prompt is not None else 0
    em = EmulatedRanks(torch, device_block, F, Lv, Lt, nranks)
    xs = em.split(x)
    outs = [torch.empty_like(t) for t in xs]
    em.block_forward(xs, prompt, outs, add_residual)
    return torch.cat(outs, dim=1)


# ---------------------------------------------------------------------------
# Sequence-parallel model step: ToyDenoiser.forward over P ranks
# ---------------------------------------------------------------------------

class FrameReshard:
    """Frame-wise -> spatial reshard of the embedded tokens (alltoall_reshard,
    executor.py:252-287, spatial axis): this rank embedded the frames
    round_robin_frames(F, P)[rank] = rank, rank + P, ... (executor.py:194-196)
    and every peer r needs rows [vb[r], vb[r+1]) of each. CUDA pack / unpack
    (vc_sp_reshard_*) around one all-to-all; the resident [F, vc_rank, D]
    equals allgather_then_shard (executor.py:290-308) exactly."""

    def __init__(self, torch, frames, visual_len, dim, heads, nranks, rank):
        self.torch, self.F, self.Lv, self.D, self.P, self.rank = torch, frames, visual_len, dim, nranks, rank
        self.plan = _lib.SpPlan(_lib.shape(frames, visual_len, 0, dim, heads, "bf16"), nranks, rank)
        lib = _lib.load()
        self.counts = {k: [int(lib.vc_sp_reshard_elems(C.byref(self.plan), i, r)) for r in range(nranks)]
                       for i, k in enumerate(("send", "recv"))}
        if min(self.counts["send"] + self.counts["recv"]) < 0:
            raise ValueError(lib.vc_last_error().decode())
        self.vb = contiguous_bounds(visual_len, nranks)
        self.send = torch.empty(max(sum(self.counts["send"]), 1), dtype=torch.float32, device="cuda")
        self.recv = torch.empty(max(sum(self.counts["recv"]), 1), dtype=torch.float32, device="cuda")

    @property
    def frames(self):
        return list(range(self.rank, self.F, self.P))

    def pack(self, local_frames):
        lib = _lib.load()
        _lib.check(lib.vc_sp_reshard_pack(C.byref(self.plan), _lib.ptr(local_frames), _lib.ptr(self.send),
                                          _lib.stream_ptr(self.torch)), "reshard pack")

    def unpack(self, resident):
        lib = _lib.load()
        _lib.check(lib.vc_sp_reshard_unpack(C.byref(self.plan), _lib.ptr(self.recv), _lib.ptr(resident),
                                            _lib.stream_ptr(self.torch)), "reshard unpack")

    def __call__(self, local_frames, exchange):
        """local_frames [len(frames), Lv, D] fp32 -> resident [F, vc_rank, D] fp32."""
        resident = self.torch.empty((self.F, self.vb[self.rank + 1] - self.vb[self.rank], self.D),
                                    dtype=self.torch.float32, device="cuda")
        self.pack(local_frames)
        if isinstance(exchange, LoggedExchange):
            exchange.stage = "reshard"
            exchange.payload = None
            exchange.bpe, bpe = 4, exchange.bpe
        exchange.all_to_all(self.recv[:sum(self.counts["recv"])], self.send[:sum(self.counts["send"])],
                            self.counts["recv"], self.counts["send"])
        if isinstance(exchange, LoggedExchange):
            exchange.bpe = bpe
        self.unpack(resident)
        return resident


def embed_frames_local(torch, model, lat_dev, t, frames):
    """ToyDenoiser.embed_frame (model.py:303-314) for the given frames -> [n, Lv, D] fp32."""
    from .numerics import to_device_f32
    F, h, w, c = lat_dev.shape
    p = model.spec.patch
    Lv = -(-h // p) * -(-w // p)
    out = torch.empty((len(frames), Lv, model.dim), dtype=torch.float32, device="cuda")
    w_in = to_device_f32(torch, model.w_in)
    lib = _lib.load()
    for i, f in enumerate(frames):
        _lib.check(lib.vc_embed_frames(_lib.ptr(lat_dev[f:f + 1]), _lib.ptr(w_in), _lib.ptr(out[i:i + 1]), 1, f,
                                       h, w, c, p, model.dim, float(t), _lib.stream_ptr(torch)), "embed frame")
    return out


def embed_rows(torch, model, lat_dev, t, tok0, ntok):
    """Rows [tok0, tok0+ntok) of every frame of ToyDenoiser.embed_frame
    (model.py:303-314) -> [F, ntok, D] fp32. Position-wise, so a rank embeds
    exactly its own rows: no frame-wise encode + all-to-all reshard
    (executor.py:535-559) is needed."""
    from .numerics import to_device_f32
    F, h, w, c = lat_dev.shape
    x = torch.empty((F, ntok, model.dim), dtype=torch.float32, device="cuda")
    w_in = to_device_f32(torch, model.w_in)
    lib = _lib.load()
    _lib.check(lib.vc_embed_frames_rows(_lib.ptr(lat_dev), _lib.ptr(w_in), _lib.ptr(x), F, 0, tok0, ntok, h, w, c,
                                        model.spec.patch, model.dim, float(t), _lib.stream_ptr(torch)), "embed rows")
    return x


def unembed(torch, model, x_full, h, w, c):
    """ToyDenoiser.forward's output projection + crop (model.py:331-333)."""
    from .numerics import to_device_f32
    F = x_full.shape[0]
    eps = torch.empty((F, h, w, c), dtype=torch.float32, device="cuda")
    w_out = to_device_f32(torch, model.w_out)
    lib = _lib.load()
    _lib.check(lib.vc_unembed_frames(_lib.ptr(x_full), _lib.ptr(w_out), _lib.ptr(eps), F, h, w, c,
                                     model.spec.patch, model.dim, _lib.stream_ptr(torch)), "unembed")
    return eps


def emulate_reshard(torch, reshards, locals_):
    """FrameReshard over P virtual ranks on one GPU: pack everywhere, the
    all-to-all as block copies with the product's per-peer counts, unpack."""
    P = len(reshards)
    for r, rs in enumerate(reshards):
        rs.pack(locals_[r])
    for dst in range(P):
        pieces = []
        for src in range(P):
            off = sum(reshards[src].counts["send"][:dst])
            pieces.append(reshards[src].send[off:off + reshards[src].counts["send"][dst]])
        torch.cat(pieces, out=reshards[dst].recv[:sum(reshards[dst].counts["recv"])])
    out = []
    for r, rs in enumerate(reshards):
        res = torch.empty((rs.F, rs.vb[r + 1] - rs.vb[r], rs.D), dtype=torch.float32, device="cuda")
        rs.unpack(res)
        out.append(res)
    return out


def emulate_sp_model_forward(torch, model, latents, t, prompt, nranks, embed="rows"):
    """ToyDenoiser.forward (bf16) over P virtual ranks: each rank embeds its
    rows, the blocks run sequence-parallel with the residual fused, the final
    all-gather (executor.py:683-693) becomes a concatenation, and the
    replicated unembed runs once."""
    from .model import device_block
    from .numerics import to_device_f32
    lat = to_device_f32(torch, latents)
    pr = to_device_f32(torch, prompt)
    F, h, w, c = lat.shape
    p = model.spec.patch
    Lv = -(-h // p) * -(-w // p)
    dbs = [device_block(torch, b, model.heads, "bf16") for b in model.blocks]
    em = EmulatedRanks(torch, dbs[0], F, Lv, pr.shape[0], nranks)
    if embed == "frames":  # frame-wise embed on each rank + the reshard (executor.py:535-559)
        rss = [FrameReshard(torch, F, Lv, model.dim, model.heads, nranks, r) for r in range(nranks)]
        xs = emulate_reshard(torch, rss, [embed_frames_local(torch, model, lat, t, rs.frames) for rs in rss])
    else:
        xs = [embed_rows(torch, model, lat, t, em.vb[r], em.vb[r + 1] - em.vb[r]) for r in range(nranks)]
    for db in dbs:
        em.block_forward(xs, pr, xs, add_residual=True, device_block=db)
    return unembed(torch, model, torch.cat(xs, dim=1).contiguous(), h, w, c)


def sp_model_forward(torch, model, latents, t, prompt, spb_cache, exchange, rank, nranks, group=None,
                     embed="rows"):
    """ToyDenoiser.forward on this rank of a P-rank job (torchrun + NCCL):
    embed own rows -> depth x SPBlock.forward (residual fused, in place) ->
    all-gather the rows (executor.py:683-693) -> unembed. Every rank returns
    the full eps [F, h, w, c] (the reference's replicated output head)."""
    import torch.distributed as dist

    from .model import device_block
    from .numerics import to_device_f32
    lat = to_device_f32(torch, latents)
    pr = to_device_f32(torch, prompt)
    F, h, w, c = lat.shape
    p = model.spec.patch
    Lv = -(-h // p) * -(-w // p)
    dbs = [device_block(torch, b, model.heads, "bf16") for b in model.blocks]
    key = (F, Lv, pr.shape[0], nranks, rank)
    if key not in spb_cache:
        spb_cache[key] = SPBlock(torch, dbs[0], F, Lv, pr.shape[0], nranks, rank)
    spb = spb_cache[key]
    lo, hi = spb.local_rows
    if embed == "frames":  # the reference's stage 1-2: frame-wise embed, then the reshard (executor.py:535-559)
        rs = FrameReshard(torch, F, Lv, model.dim, model.heads, nranks, rank)
        x = rs(embed_frames_local(torch, model, lat, t, rs.frames), exchange)
    else:  # position-wise embed of the own rows: the same residents without a collective
        x = embed_rows(torch, model, lat, t, lo, hi - lo)
    for bi, db in enumerate(dbs):
        spb.db = db
        spb.forward(x, pr, x, exchange, add_residual=True, stage_prefix=f"block{bi}")
    # all-gather the rows (uneven shards: pad to the largest, gather, trim)
    vmax = max(spb.vb[r + 1] - spb.vb[r] for r in range(nranks))
    pad = torch.zeros((F, vmax, model.dim), dtype=torch.float32, device="cuda")
    pad[:, :hi - lo] = x
    allx = torch.empty((nranks, F, vmax, model.dim), dtype=torch.float32, device="cuda")
    if isinstance(exchange, LoggedExchange):  # executor.py:683-693 "gather" (fp32 rows here)
        exchange.log.record("gather", "allgather", nranks, exchange.placement, pad.numel() * 4,
                            F * (hi - lo) * model.dim * 4)
    dist.all_gather_into_tensor(allx, pad, group=group)
    full = torch.cat([allx[r, :, :spb.vb[r + 1] - spb.vb[r]] for r in range(nranks)], dim=1).contiguous()
    return unembed(torch, model, full, h, w, c)


# ---------------------------------------------------------------------------
# bench.py --gpus N (torchrun, one rank per GPU)
# ---------------------------------------------------------------------------

def time_exchanges(torch, spb, ex, reps=5):
    """Each branch's two all-to-alls timed ALONE (not overlapped), with CUDA
    events on the current stream around a blocking all_to_all_single (the
    current stream waits for NCCL's stream, so the interval is the
    collective). Returns {name: ms} per rank."""
    bc = branch_counts(spb.counts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {}
    for b, bn in ((0, "spatial"), (1, "fullseq")):
        for send, recv, sc, rc, tag in (("send1", "recv1", "send1", "recv1", "a2a1"),
                                        ("send2", "recv2", "send2", "recv2", "a2a2")):
            args = (_half(getattr(spb, recv), b), _half(getattr(spb, send), b), bc[rc], bc[sc])
            ex.all_to_all(*args)  # warm
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                ex.all_to_all(*args)
            e1.record()
            torch.cuda.synchronize()
            out[f"{bn}_{tag}"] = e0.elapsed_time(e1) / reps
    return out


def bench_sp(args, torch, world, rank, local, CONFIGS, METRIC, algorithmic_flops, load_peaks, tensor_peak,
             ClockSampler, cpu_slices, time_slices, slice_sample_text, cpu_cores, stage_profile=None):
    import json
    import torch.distributed as dist

    from .model import DeviceBlock
    from .numerics import SeededRng
    from .model import BlockParams

    import os
    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531"), ("RANK", "0"), ("WORLD_SIZE", "1")):
        os.environ.setdefault(k, v)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    F, Lv, Lt, D, H, name = CONFIGS[args.config]
    blk = BlockParams.init(SeededRng(2025).split(1000), D)
    db = DeviceBlock(torch, blk, H, "bf16")
    # head-parallel (the reference's default) unless P does not divide H or
    # gather mode is asked for (executor.py:462-466)
    mode = getattr(args, "sp_mode", "head_parallel")
    if mode == "gather" or H % world != 0:
        mode = "gather"
        spb = SPGatherBlock(torch, db, F, Lv, Lt, world, rank)
    else:
        spb = SPBlock(torch, db, F, Lv, Lt, world, rank)
    lo, hi = spb.local_rows
    g = torch.Generator(device="cuda").manual_seed(2025)
    x_full = torch.randn((F, Lv, D), device="cuda", generator=g)  # same on every rank (same seed)
    prompt = torch.randn((Lt, D), device="cuda", generator=g)
    x_local = x_full[:, lo:hi].contiguous()
    del x_full
    out = torch.empty_like(x_local)
    ex = TorchExchange()
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3)):
        spb.forward(x_local, prompt, out, ex)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            spb.forward(x_local, prompt, out, ex)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(ms.item())
    Nv = F * Lv
    value = Nv / (ms_per_step / 1e3)
    # end to end: host (pinned) local rows in, host out, per rank; the H2D of
    # step i+1 and the D2H of step i-1 run on a copy stream under the
    # forward of step i (double-buffered, as the single-GPU serving path)
    xh = [x_local.cpu().pin_memory() for _ in range(2)]
    oh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
    xd = [torch.empty_like(x_local) for _ in range(2)]
    od = [torch.empty_like(x_local) for _ in range(2)]
    cs = torch.cuda.Stream()

    def e2e_steps(n):
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            xd[0].copy_(xh[0], non_blocking=True)
            ev_in[0].record(cs)
        for i in range(n):
            b = i % 2
            if i + 1 < n:
                with torch.cuda.stream(cs):  # stream order: after the D2H of step i-1
                    xd[1 - b].copy_(xh[1 - b], non_blocking=True)
                    ev_in[1 - b].record(cs)
            stream.wait_event(ev_in[b])
            spb.forward(xd[b], prompt, od[b], ex)
            ev_done[b].record(stream)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_done[b])
                oh[b].copy_(od[b], non_blocking=True)
        stream.wait_stream(cs)

    e2e_steps(3)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    e2e_steps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    # per-stage device time of this rank's kernels (untimed pass; the waits for
    # the exchanges happen between the stage calls and are not counted)
    stages_ms = None
    if stage_profile is not None:
        stages_ms = stage_profile(torch, _lib.load(), lambda: spb.forward(x_local, prompt, out, ex), 3)
    # one untimed forward with the collectives logged (executor.py:111-141 CommLog rows)
    comm = CommLog()
    spb.forward(x_local, prompt, out, LoggedExchange(ex, comm, world, bpe=2))
    torch.cuda.synchronize()
    # the exchanges alone (untimed pass): NVLink GB/s per rank, max time over ranks
    a2a = {"mode": mode, "comm_log": [[*e.key(), e.payload_bytes] for e in comm.events],
           "comm_log_fields": ["stage", "collective", "group_size", "placement", "bytes_per_device (as sent)",
                               "payload_bytes (reference payload: no head-dim padding)"]}
    if mode == "head_parallel":
        t = time_exchanges(torch, spb, ex)
        tt = torch.tensor([t[k] for k in sorted(t)], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = dict(zip(sorted(t), tt.tolist()))
        bc = branch_counts(spb.counts)
        ref = branch_counts(exchange_counts(F, Lv, H, D, world, rank, padded=False))
        for k, ms_k in t.items():
            tag = "send1" if k.endswith("a2a1") else "send2"
            # bytes leaving this rank over NVLink (its own block stays local)
            wire = 2 * (sum(bc[tag]) - bc[tag][rank])
            alg = 2 * (sum(ref[tag]) - ref[tag][rank])
            gbs = (lambda b: b / (ms_k / 1e3) / 1e9 if ms_k > 0 else 0.0)  # noqa: E731
            a2a[k] = {"ms": ms_k, "nvlink_bytes_per_rank": wire, "nvlink_gbs": gbs(wire),
                      "algorithmic_bytes_per_rank": alg, "algorithmic_gbs": gbs(alg)}
        a2a["note"] = ("each all-to-all timed alone (blocking, CUDA events, max over ranks); in the block "
                       "step they overlap attention (sp.run_stages). nvlink_bytes = what this rank sends to "
                       "its peers as laid out (head dim padded 66 -> 80); algorithmic = the reference's "
                       "payload (executor.py:344-347, :395-412). The own block never enters the exchange buffers "
                       "(stage 1 / 2 write it where stage 2 / 3 read it): at 1 rank there is no collective.")
    else:  # bf16 bytes sent per rank: own slot to every peer
        a2a["bytes_sent_per_rank_per_step"] = 2 * spb.slot * (world - 1)
    flops = sum(algorithmic_flops(F, Lv, Lt, D, H).values())
    peaks = load_peaks()
    clocks = clk.summary()
    all_clocks = [None] * world
    dist.all_gather_object(all_clocks, clocks)
    # the bound for every rank: burst only if every rank stayed at its max clock
    peak_kinds = [tensor_peak(peaks, c) for c in all_clocks]
    peak, peak_kind = min(peak_kinds)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        fs = cpu_slices(args.config)
        ts = time_slices(fs, 2)
        cpu = {"value": 2 * Lv / sum(ts), "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
               "sample": slice_sample_text(args.config, 2)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (torch.randn inputs, SeededRng random-init 2B-shape weights)",
            "config": {"workload": name, "frames": F, "visual_len": Lv, "text_len": Lt, "dim": D, "heads": H,
                       "tokens_per_step": Nv,
                       "parallelism": (f"sequence parallel sp{world} (spatial shard axis, "
                                       + ("head-parallel a2a" if mode == "head_parallel" else "K/V all-gather")
                                       + ", NCCL)"),
                       "l2": "inputs larger than L2 on every rank"},
            "roofline": {"bound": "tensor", "kernel": "whole block (per GPU)",
                         "achieved": flops / world / (ms_per_step / 1e3) / 1e12, "peak": peak,
                         "unit": "TFLOP/s", "frac": flops / world / (ms_per_step / 1e3) / 1e12 / peak,
                         "traffic": None, "peak_kind": peak_kind},
            "a2a": a2a,
            "stage_ms": stages_ms,
            "cpu_baseline": cpu,
            "e2e": {"value": Nv / (float(e2e.item()) / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(xh[0].numel() * 4) * world, "d2h_bytes_per_step": int(oh[0].numel() * 4) * world},
            "clocks": clocks,
            "clocks_per_rank": all_clocks,
            "gpu_launches": spb.launches_per_forward() * args.steps,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()

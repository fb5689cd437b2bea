"""Re-pricing the sequence-parallel block with measured B200 numbers
("re-price the planner with measured B200 kernel and NVLink
numbers, ClusterSpec with B200 values").

The reference prices collectives with an alpha-beta model
(`cluster.py:97-118`, replayed by `comm_plan_time` executor.py:776-783) on a
`ClusterSpec` (cluster.py:24-57) whose defaults describe an A100 cluster. This
module gives:

* `B200Spec` — the same fields and SI units with this pool's B200 values: the
  measured sustained bf16 rate and HBM size, the measured pinned host copy
  rate (bench e2e), NVLink 5 per-direction bandwidth (nominal: NCCL across
  GPUs is not measurable on the one-GPU pool; bench.py --sp reports the
  world-1 exchange times, which are local copies) and an assumed NCCL
  latency.
  `as_cluster_kwargs()` builds the reference's own `ClusterSpec(**kwargs)`.
* `alltoall_time` — the reference's all-to-all formula (cluster.py:112-118).
* `price_sp_block` — one block forward on P ranks of this implementation's
  head-parallel schedule: the MEASURED single-GPU per-stage times
  (`bench.py` block.stage_ms, CUDA events) divided over the ranks the way the
  work divides (local rows for LN / QKV / temporal / O, H/P heads for the two
  attentions), plus the two per-branch all-to-alls priced with the exact byte
  counts this implementation sends (`sp.exchange_counts`: q, k, v with the
  head dim padded to 80), either fully exposed or overlapped the way
  `sp.run_stages` schedules them (both a2a #1 under the temporal branch and
  the spatial attention, a2a #2 of the spatial branch under the
  full-sequence attention).

These are PRICED numbers (a model), not measurements; profiles/ labels them
so. Pure host code: no GPU needed.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass

from .sp import contiguous_bounds, exchange_counts, head_pad


@dataclass(frozen=True)
class B200Spec:
    """ClusterSpec fields (cluster.py:24-57), SI units, for one 8x B200 node."""
    nodes: int = 1
    devices_per_node: int = 8
    intra_bw: float = 900e9          # NVLink 5 / NVSwitch, per GPU per direction (nominal)
    inter_bw: float = 50e9           # one 400 Gb/s NIC per GPU (nominal)
    h2d_bw: float = 57.6e9           # measured: pinned copies in bench e2e (profiles/r01)
    offload_exposed_bw: float = 0.9e9  # reference default (offload is out of scope)
    device_mem: float = 180e9        # HBM3e per B200
    host_mem: float = 2e12
    compute_rate: float = 1386.1e12  # measured sustained dense bf16 (MEASURED_PEAKS.json)
    alpha: float = 10e-6             # assumed NCCL all-to-all latency per peer hop
    attention_heads: int = 24

    def as_cluster_kwargs(self) -> dict:
        return asdict(self)


def alltoall_time(p: int, bytes_per_device: float, bw: float, alpha: float) -> float:
    """cluster.py:112-118: each device re-deals its b bytes, 1/P stay local."""
    if p < 1:
        raise ValueError(f"group size must be >= 1, got {p}")
    if p == 1:
        return 0.0
    return alpha * (p - 1) + (p - 1) / p * bytes_per_device / bw


# stage names of bench.py's block.stage_ms and how each divides over P ranks
_ROW_STAGES = ("ln", "qkv_gemm", "attn_temporal", "oproj_gemm")   # local rows (1/P)
_HEAD_STAGES = ("attn_spatial", "attn_fullseq", "text_kv_gemm")   # H/P heads (1/P)


def price_sp_block(stage_ms: dict, frames: int, visual_len: int, text_len: int, dim: int, heads: int,
                   p: int, spec: B200Spec = B200Spec(), overlap: bool = True,
                   sp_overhead_ms: float = 0.0) -> dict:
    """Priced time of one block forward on P ranks (slowest rank), from the
    measured single-GPU stage times. sp_overhead_ms: the SP path's extra
    layout passes (exchange-buffer unpacks) over the FULL data at one rank;
    a rank unpacks only its peers' share of its 1/P. Returns ms per block, the exchange bytes
    per rank and the exposed communication."""
    if heads % p:
        raise ValueError(f"head-parallel pricing needs P | H ({p} does not divide {heads})")
    vb = contiguous_bounds(visual_len, p)
    rows_max = max(vb[r + 1] - vb[r] for r in range(p))
    row_share = rows_max / visual_len          # the slowest rank's share of the rows
    head_share = 1.0 / p
    compute = {k: v * (row_share if k in _ROW_STAGES else head_share if k in _HEAD_STAGES else 1.0)
               for k, v in stage_ms.items()}
    # slowest rank's bytes: the one with the most rows sends/receives most
    r_max = max(range(p), key=lambda r: vb[r + 1] - vb[r])
    c = exchange_counts(frames, visual_len, heads, dim, p, r_max)
    # bytes per branch per device as the reference's alpha-beta term counts
    # them (own block included; (p-1)/p of it crosses the links): the counts
    # as laid out exclude the own block, which has the size of any peer's
    other = (r_max + 1) % p
    a2a1 = (sum(c["send1"]) + c["send1"][other]) * 2.0 / 2   # bf16, branch-major halves
    a2a2 = (sum(c["recv2"]) + c["recv2"][other]) * 2.0 / 2
    t1 = alltoall_time(p, a2a1, spec.intra_bw, spec.alpha) * 1e3   # ms per branch
    t2 = alltoall_time(p, a2a2, spec.intra_bw, spec.alpha) * 1e3
    comm = 2 * (t1 + t2)
    if not overlap or p == 1:
        exposed = comm
    else:
        # sp.run_stages (NCCL runs its collectives one after another on its
        # own stream; compute on the main stream):
        #   both a2a #1 start after the QKV GEMM; the temporal branch runs under them
        #   spatial attention once a2a#1(spatial) landed; a2a#2(spatial) after it
        #   full-seq attention once a2a#1(full seq) landed; a2a#2(full seq) after it
        #   the O projection once both a2a #2 landed
        tm = compute.get("attn_temporal", 0.0)
        sp_att, fs_att = compute.get("attn_spatial", 0.0), compute.get("attn_fullseq", 0.0)
        net = 2 * t1                      # NCCL stream busy until both a2a #1 are done
        a1_sp, a1_fs = t1, 2 * t1
        sp_end = max(tm, a1_sp) + sp_att
        a2_sp = max(sp_end, net) + t2
        fs_end = max(sp_end, a1_fs) + fs_att
        a2_fs = max(fs_end, a2_sp) + t2
        exposed = a2_fs - (tm + sp_att + fs_att)  # the critical path beyond the compute it overlaps
    # the unpacks of the peers' share ((p-1)/p of this rank's 1/p of the data)
    layout = sp_overhead_ms * row_share * (p - 1) / p if p > 1 else 0.0
    total = sum(compute.values()) + layout + exposed
    return {"p": p, "ms": total, "compute_ms": sum(compute.values()) + layout, "comm_ms": comm,
            "exposed_comm_ms": exposed, "a2a1_bytes_per_branch": a2a1, "a2a2_bytes_per_branch": a2a2}


def price_scaling(stage_ms: dict, frames: int, visual_len: int, text_len: int, dim: int, heads: int,
                  ps=(1, 2, 4, 8), spec: B200Spec = B200Spec(), overlap: bool = True,
                  sp_overhead_ms: float = 0.0) -> list:
    """Priced strong scaling: tokens/s and T1 / (P * TP) per P."""
    rows = []
    t1 = None
    for p in ps:
        if heads % p:
            continue
        r = price_sp_block(stage_ms, frames, visual_len, text_len, dim, heads, p, spec, overlap, sp_overhead_ms)
        t1 = r["ms"] if p == 1 else t1
        r["tokens_per_s"] = frames * visual_len / (r["ms"] / 1e3)
        r["efficiency"] = (t1 / (p * r["ms"])) if t1 else None
        rows.append(r)
    return rows

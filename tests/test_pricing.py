"""The B200 re-pricing of the SP block (a model, not a
measurement): the all-to-all formula equals the reference's, the spec builds
the reference's own ClusterSpec, and the priced scaling behaves."""
import importlib
import os
import sys

import pytest

from paper_2501_08453_b200 import pricing

REF = "/root/reference/pkg/src"
STAGES = {"ln": 0.037, "qkv_gemm": 0.868, "text_kv_gemm": 0.025, "attn_spatial": 0.397,
          "attn_temporal": 0.079, "attn_fullseq": 3.481, "oproj_gemm": 0.248}   # profiles/r01 config 2


def _ref_cluster():
    if not os.path.isdir(REF):
        pytest.skip("reference not mounted")
    sys.path.insert(0, REF)
    try:
        return importlib.import_module("spsim.cluster")
    finally:
        sys.path.remove(REF)


def test_alltoall_matches_reference_formula():
    cl = _ref_cluster()
    for p, b, bw, a in [(1, 1e6, 9e11, 1e-5), (2, 3.3e8, 9e11, 1e-5), (8, 7.1e7, 3e11, 5e-6), (3, 1.0, 1.0, 0.0)]:
        assert pricing.alltoall_time(p, b, bw, a) == pytest.approx(cl.alltoall_time(p, b, bw, a), rel=1e-15)


def test_spec_builds_reference_cluster_spec():
    cl = _ref_cluster()
    spec = cl.ClusterSpec(**pricing.B200Spec().as_cluster_kwargs())
    assert spec.total_devices == 8 and spec.intra_bw == 900e9 and spec.compute_rate == pytest.approx(1386.1e12)


def test_priced_scaling_config3_shape():
    rows = pricing.price_scaling(STAGES, 40, 1350, 256, 1584, 24, ps=(1, 2, 3, 4, 6, 8))
    assert [r["p"] for r in rows] == [1, 2, 3, 4, 6, 8]
    assert rows[0]["exposed_comm_ms"] == 0.0 and rows[0]["efficiency"] == pytest.approx(1.0)
    for a, b in zip(rows, rows[1:]):
        assert b["ms"] < a["ms"]                      # more ranks, less time per block
        assert 0.0 < b["efficiency"] <= 1.0 + 1e-12
    # overlap never prices slower than the fully exposed exchange
    for p in (2, 4, 8):
        o = pricing.price_sp_block(STAGES, 40, 1350, 256, 1584, 24, p)
        x = pricing.price_sp_block(STAGES, 40, 1350, 256, 1584, 24, p, overlap=False)
        assert o["ms"] <= x["ms"] and o["comm_ms"] == x["comm_ms"]


def test_pricing_rejects_p_not_dividing_heads():
    with pytest.raises(ValueError):
        pricing.price_sp_block(STAGES, 4, 64, 32, 256, 4, 3)

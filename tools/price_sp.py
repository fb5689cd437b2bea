"""Priced strong scaling of the SP block from this round's measured stage
times (paper_2501_08453_b200.pricing; a MODEL, not a measurement — the pool
has one GPU per box).  Writes profiles/r02/sp_pricing.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_08453_b200 import pricing  # noqa: E402

SHAPES = {2: (16, 1350, 256, 1584, 24, "profiles/r02/configs/bench_config2.json"),
          4: (160, 1350, 256, 1584, 24, "profiles/r02/configs/bench_cfg4.json"),
          5: (64, 256, 256, 3072, 24, "profiles/r02/configs/bench_cfg5.json")}
out = {"what": "PRICED (alpha-beta model on measured single-GPU stage times), not measured: "
               "paper_2501_08453_b200/pricing.py; spec = B200Spec (NVLink 900 GB/s nominal, alpha 10 us assumed)",
       "spec": pricing.B200Spec().as_cluster_kwargs(), "configs": {}}
# the SP path's unpack passes over the FULL config-2 data (sp_unpack1 spatial
# 0.189 + full sequence 0.130 + sp_unpack2 0.059 ms: the stage profile of
# bench.py --sp at P = 1 before the own block bypassed the buffers, this
# round); a rank now unpacks only its peers' share (pricing.price_sp_block);
# scaled to the other configs by activation size (memory-bound copies)
SP_UNPACK_FULL_CFG2 = 0.189 + 0.130 + 0.059
for cfg, (F, Lv, Lt, D, H, path) in SHAPES.items():
    stages = json.load(open(os.path.join(ROOT, path)))["block"]["stage_ms"]
    ovh = SP_UNPACK_FULL_CFG2 * (F * Lv * D) / (16 * 1350 * 1584)
    out["configs"][f"config{cfg}"] = {
        "stage_ms_measured_1gpu": stages, "sp_unpack_full_data_ms": ovh,
        "overlapped": pricing.price_scaling(stages, F, Lv, Lt, D, H, ps=(1, 2, 3, 4, 6, 8), sp_overhead_ms=ovh),
        "exposed": pricing.price_scaling(stages, F, Lv, Lt, D, H, ps=(1, 2, 3, 4, 6, 8), overlap=False,
                                         sp_overhead_ms=ovh),
    }
out["sp_unpack_full_data_cfg2_ms"] = SP_UNPACK_FULL_CFG2
json.dump(out, open(os.path.join(ROOT, "profiles/r02/sp_pricing.json"), "w"), indent=1)
for k, v in out["configs"].items():
    print(k, [(r["p"], round(r["ms"], 3), round(r["efficiency"], 3)) for r in v["overlapped"]])

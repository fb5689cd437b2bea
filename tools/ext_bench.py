"""Time the north-star extended block (AdaLN + QK-RMSNorm/3D RoPE + gated GELU
FFN, vc_ext_block_forward) next to the reference-semantics block on the same
shape, with per-stage device times.  Not the headline bench (bench.py is);
the numbers go to profiles/r01/ext/.

    python tools/ext_bench.py [--config 2] [--steps 10] [--warmup 3]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--mlp-ratio", type=float, default=2.0)
    a = ap.parse_args()
    import torch
    import paper_2501_08453_b200 as vc
    from paper_2501_08453_b200 import _lib
    from paper_2501_08453_b200.model import block_forward_device
    from paper_2501_08453_b200.vchitect import VchitectBlock, VchitectExtParams

    F, Lv, Lt, D, H, name = bench.CONFIGS[a.config]
    grid = {1350: (30, 45), 256: (16, 16), 64: (8, 8)}[Lv]
    Nv = F * Lv
    params = VchitectExtParams.init(vc.SeededRng(2025), D, H, a.mlp_ratio)
    blk = VchitectBlock(params, H, grid)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn((F, Lv, D), device="cuda", generator=g)
    prompt = torch.randn((Lt, D), device="cuda", generator=g)
    out = torch.empty_like(x)
    lib = _lib.load()

    def ext():
        blk.forward_device(x, prompt, 500, out)

    def base():
        block_forward_device(torch, blk.db, x, prompt, out, True)

    res = {}
    for nm, fn in (("reference_block", base), ("extended_block", ext)):
        for _ in range(max(a.warmup, 3)):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        res[nm] = {"ms_per_step": ms, "tokens_per_s": Nv / (ms / 1e3),
                   "stage_ms": bench.stage_profile(torch, lib, fn, 3)}
    fl = bench.algorithmic_flops(F, Lv, Lt, D, H)
    dff = blk.ffn_dim
    ffn = 2.0 * 2 * Nv * D * dff
    peaks = bench.load_peaks()
    st = res["extended_block"]["stage_ms"]
    ffn_ms = st.get("ffn1_gemm", 0) + st.get("ffn2_gemm", 0)
    line = {
        "what": "extended block (north-star AdaLN + QK-RMSNorm/3D RoPE + gated GELU FFN), parity unpinned",
        "config": {"workload": name, "grid": grid, "ffn_dim": dff, "dtype": "bf16"},
        **res,
        "ffn_tflops": ffn / (ffn_ms / 1e3) / 1e12 if ffn_ms else None,
        "ffn_frac_sustained": ffn / (ffn_ms / 1e3) / 1e12 / peaks["tc_sus"] if ffn_ms else None,
        "extended_block_tflops_algorithmic": (sum(fl.values()) + ffn) / (res["extended_block"]["ms_per_step"] / 1e3) / 1e12,
        "launches_per_forward": lib.vc_ext_block_launches(C.byref(blk.shape(F, Lv, Lt))),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

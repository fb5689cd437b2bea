"""Run the bf16 block forward a few times on cuda:0 (profiling driver)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2501_08453_b200.model import block_forward_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--dtype", default="bf16")
a = ap.parse_args()
F, Lv, Lt, D, H, _ = CONFIGS[a.config]
db, x, prompt = make_inputs(torch, a.config, D, H, a.dtype)
out = torch.empty_like(x)
for _ in range(a.iters):
    block_forward_device(torch, db, x, prompt, out, False)
torch.cuda.synchronize()
assert torch.isfinite(out).all().item()
print("ok", float(out.abs().mean()))

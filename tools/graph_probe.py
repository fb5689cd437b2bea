"""Block forward launched directly vs replayed from a captured CUDA graph
(config 2, 10 steps each, interleaved 3 times; CUDA events on the stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2501_08453_b200.model import block_forward_device  # noqa: E402

F, Lv, Lt, D, H, _ = CONFIGS[2]
db, x, prompt = make_inputs(torch, 2, D, H, "bf16")
out = torch.empty_like(x)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        block_forward_device(torch, db, x, prompt, out, False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        block_forward_device(torch, db, x, prompt, out, False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(3):
        for mode in ("direct", "graph"):
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(10):
                if mode == "graph":
                    g.replay()
                else:
                    block_forward_device(torch, db, x, prompt, out, False)
            e1.record(s)
            torch.cuda.synchronize()
            print(mode, round(e0.elapsed_time(e1) / 10, 4), "ms")

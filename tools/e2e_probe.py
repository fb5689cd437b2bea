"""Probe the end-to-end (pinned host in/out) serving path: raw PCIe copy
rates and the overlap achieved by vc_block_forward_host_batched."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2501_08453_b200.model import block_forward_device, block_forward_host_stream  # noqa: E402


def timed(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


F, Lv, Lt, D, H, _ = CONFIGS[2]
db, x, prompt, blk = make_inputs(torch, 2, D, H, "bf16", return_block=True)
nb = x.numel() * 4
xh = x.cpu().pin_memory()
yh = torch.empty_like(xh).pin_memory()
xd = torch.empty_like(x)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2d = timed(lambda: xd.copy_(xh, non_blocking=True))
d2h = timed(lambda: yh.copy_(x, non_blocking=True))


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(x, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


bi = timed(both)
out = torch.empty_like(x)
comp = timed(lambda: block_forward_device(torch, db, x, prompt, out, False))
print(f"bytes {nb / 1e6:.1f} MB: H2D {h2d:.3f} ms ({nb / h2d / 1e6:.1f} GB/s), D2H {d2h:.3f} ms "
      f"({nb / d2h / 1e6:.1f} GB/s), both concurrently {bi:.3f} ms, block compute {comp:.3f} ms")
ph = prompt.cpu().pin_memory()
for n in (2, 4, 8, 16):
    xs = [xh if i % 2 == 0 else xh.clone().pin_memory() for i in range(n)]
    ys = [torch.empty_like(xh).pin_memory() for _ in range(n)]
    ms = timed(lambda: block_forward_host_stream(blk, xs, ph, H, ys, dtype="bf16"), reps=2) / n
    print(f"host stream n={n}: {ms:.3f} ms/step -> {F * Lv / ms / 1e3:.3f} M tok/s")

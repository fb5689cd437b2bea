"""Probe the gap between the timed block loop and the per-stage sum:
back-to-back forwards vs forwards separated by a host sync vs the stage
profiler, each timed with CUDA events on the launching stream."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2501_08453_b200 import _lib
from paper_2501_08453_b200.model import block_forward_device

F, Lv, Lt, D, H, _ = bench.CONFIGS[2]
db, x, prompt = bench.make_inputs(torch, 2, D, H, "bf16")
out = torch.empty_like(x)
lib = _lib.load()
fwd = lambda: block_forward_device(torch, db, x, prompt, out, False)
for _ in range(3): fwd()
torch.cuda.synchronize()
n = 20
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
for rep in range(2):
    ev[0].record()
    for i in range(n):
        fwd(); ev[i + 1].record()
    torch.cuda.synchronize()
    t = [ev[i].elapsed_time(ev[i + 1]) for i in range(n)]
    print("back-to-back  mean %.3f  min %.3f  max %.3f" % (sum(t) / n, min(t), max(t)))
    t = []
    for i in range(n):
        ev[0].record(); fwd(); ev[1].record(); torch.cuda.synchronize()
        t.append(ev[0].elapsed_time(ev[1]))
    print("synced        mean %.3f  min %.3f  max %.3f" % (sum(t) / n, min(t), max(t)))
    for gap_us in (20, 100):
        t = []
        for i in range(n):
            ev[0].record(); torch.cuda._sleep(int(gap_us * 1965)); ev[1].record(); fwd(); ev[2].record()
            t.append(ev[1].elapsed_time(ev[2]))
        torch.cuda.synchronize()
        t = [ev[1].elapsed_time(ev[2])]
        print("sleep %d us before each fwd: last %.3f" % (gap_us, t[0]))
    st = bench.stage_profile(torch, lib, fwd, 5)
    print("stage sum %.3f" % sum(st.values()), {k: round(v, 3) for k, v in st.items()})

"""Probe the gap between the timed block loop and the per-stage sum: host
launch cost per forward, back-to-back device time, and the same forward
replayed from a CUDA graph."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2501_08453_b200.model import block_forward_device

F, Lv, Lt, D, H, _ = bench.CONFIGS[2]
db, x, prompt = bench.make_inputs(torch, 2, D, H, "bf16")
out = torch.empty_like(x)
fwd = lambda: block_forward_device(torch, db, x, prompt, out, False)
for _ in range(3): fwd()
torch.cuda.synchronize()
# host cost per call (GPU kept busy by a long queue)
t0 = time.perf_counter(); n = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): fwd()
t1 = time.perf_counter()
e1.record(); torch.cuda.synchronize()
print("host us/call %.1f  device ms/step %.3f" % ((t1 - t0) / n * 1e6, e0.elapsed_time(e1) / n))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    fwd()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    fwd()
torch.cuda.synchronize()
for _ in range(3): g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(n): g.replay()
e1.record(); torch.cuda.synchronize()
print("graph device ms/step %.3f" % (e0.elapsed_time(e1) / n))
e0.record()
for _ in range(n): fwd()
e1.record(); torch.cuda.synchronize()
print("eager again ms/step %.3f" % (e0.elapsed_time(e1) / n))
ref = out.clone(); g.replay(); torch.cuda.synchronize()
fwd(); torch.cuda.synchronize()
print("graph == eager:", torch.equal(ref, out))

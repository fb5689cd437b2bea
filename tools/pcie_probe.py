"""Pinned host <-> device copy bandwidth on this box (the e2e leg's bound):
H2D alone, D2H alone, both at once on two streams; 137 MB = one config-2
block input (fp32 [16][1350][1584])."""
import torch

n = 16 * 1350 * 1584
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, device="cuda")
d_b = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


gb = n * 4 / 1e9
t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
t_both = timed(both)
print(f"H2D {gb / t_h2d * 1e3:.1f} GB/s ({t_h2d:.3f} ms), D2H {gb / t_d2h * 1e3:.1f} GB/s ({t_d2h:.3f} ms), "
      f"both at once {t_both:.3f} ms for {gb:.3f} GB each way ({gb / t_both * 1e3:.1f} GB/s per direction)")

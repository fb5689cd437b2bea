"""Per-CTA cost model of the tc3 attention: one wave of CTAs (sq = 1536 ->
6 x 24 heads = 144 CTAs), key length swept; run under
`ncu --metrics gpu__time_duration.sum -k regex:attn_tc3` so the kernel time
is the CTA latency. Intercept = fixed per-CTA cost, slope = per key block."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2501_08453_b200 as vc
r = np.random.default_rng(0)
H, dh, sq = 24, 66, 1536
q = r.standard_normal((sq, H * dh))
for sk in [128, 256, 512, 1024, 1350, 2048, 4096, 8192]:
    k = r.standard_normal((sk, H * dh)); v = r.standard_normal((sk, H * dh))
    for _ in range(2):
        vc.attention(q, k, v, H, dtype="bf16")
    print("sk", sk, flush=True)

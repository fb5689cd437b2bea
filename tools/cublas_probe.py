import torch, json
def t(M, N, K, reps=20):
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for _ in range(3): c = a @ b.t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): c = a @ b.t()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 2 * M * N * K / ms / 1e9
for name, (M, N, K) in {"qkv (compact N 9D)": (21600, 14256, 1584), "qkv padded N": (21600, 17280, 1584),
                        "oproj (K 3*H*80)": (21600, 1584, 5760), "oproj K 3D": (21600, 1584, 4752)}.items():
    ms, tf = t(M, N, K)
    print(f"{name}: cuBLAS {ms:.4f} ms {tf:.1f} TFLOP/s")

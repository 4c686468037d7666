"""Development: HBM ceiling of the C3 access pattern (two 50 MB input
streams, one 50 MB output stream) with torch elementwise kernels, rotating
3 buffer sets through a CUDA graph like scripts/c3_sweep.py."""
import json
import torch

n = 3 << 24  # bytes per stream (C3: 2^24 records x 3 bytes)
sets = [(torch.randint(0, 7, (n,), dtype=torch.uint8, device="cuda"),
         torch.randint(0, 7, (n,), dtype=torch.uint8, device="cuda"),
         torch.empty(n, dtype=torch.uint8, device="cuda")) for _ in range(3)]
w = [(torch.empty(n // 4, dtype=torch.int32, device="cuda"), torch.empty(n // 4, dtype=torch.int32, device="cuda"),
      torch.empty(n // 4, dtype=torch.int32, device="cuda")) for _ in range(3)]


def t(fns, reps=15):
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / len(fns))
    return sorted(ts)[len(ts) // 2]


res = {}
ms = t([lambda s=s: torch.add(s[0], s[1], out=s[2]) for s in sets] * 4)
res["add_u8_us"] = ms * 1e3
res["add_u8_TBps"] = 3 * n / (ms * 1e-3) / 1e12
ms = t([lambda s=s: torch.add(s[0], s[1], out=s[2]) for s in w] * 4)
res["add_i32_us"] = ms * 1e3
res["add_i32_TBps"] = 3 * n / (ms * 1e-3) / 1e12
ms = t([lambda s=s: s[2].copy_(s[0]) for s in sets] * 4)
res["copy_u8_TBps"] = 2 * n / (ms * 1e-3) / 1e12
print(json.dumps(res))

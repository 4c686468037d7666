"""Development: K6 timings (CUDA graph of 2 launches) for the bench's two parameter sets."""
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

n = 1 << 16
g = torch.Generator(device="cuda").manual_seed(6)
a = torch.randint(0, 3, (n,), dtype=torch.uint8, device="cuda", generator=g)
b = torch.randint(0, 3, (n,), dtype=torch.uint8, device="cuda", generator=g)
o = torch.empty(2 * n - 1, dtype=torch.uint8, device="cuda")
for q, d, nq in ((32, 3, 1), (1 << 13, 1, 409), (1 << 12, 1, 64), (1 << 7, 3, 18)):
    pm = Q.PolymulPlan(3 if q != 128 else 2, q, d + 1, nq)
    for _ in range(3):
        pm.fqt_mul(a if q != 128 else a % 2, b if q != 128 else b % 2, out=o)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            pm.fqt_mul(a, b, out=o)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 5)
    ts.sort()
    words = (n // (d + 1)) ** 2
    print(f"q={q} d={d} nq={nq}: {ts[len(ts)//2]:.4f} ms  {2 * words / ts[len(ts)//2] / 1e9:.2f} TFLOP/s-equiv")

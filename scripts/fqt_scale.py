"""Development: K6 DMMA path (q = 2^13, d = 1, n_q = 409) vs operand length."""
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

pm = Q.PolymulPlan(3, 1 << 13, 2, 409)
g = torch.Generator(device="cuda").manual_seed(6)
for lg in (14, 16, 18, 20):
    n = 1 << lg
    a = torch.randint(0, 3, (n,), dtype=torch.uint8, device="cuda", generator=g)
    b = torch.randint(0, 3, (n,), dtype=torch.uint8, device="cuda", generator=g)
    o = torch.empty(2 * n - 1, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        pm.fqt_mul(a, b, out=o)
    torch.cuda.synchronize()
    reps = 5 if lg < 20 else 2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pm.fqt_mul(a, b, out=o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    words = (n // 2) ** 2
    print(f"n=2^{lg}: {ms:.4f} ms  {2 * words / ms / 1e9:.2f} TFLOP/s useful")

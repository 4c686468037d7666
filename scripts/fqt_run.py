"""Development: one K6 chunked FQT product per param set (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

n = 1 << 16
g = torch.Generator(device="cuda").manual_seed(6)
a = torch.randint(0, 3, (n,), dtype=torch.uint8, device="cuda", generator=g)
b = torch.randint(0, 3, (n,), dtype=torch.uint8, device="cuda", generator=g)
for q, d, nq in ((32, 3, 1), (1 << 13, 1, 409)):
    pm = Q.PolymulPlan(3, q, d + 1, nq)
    for _ in range(2):
        pm.fqt_mul(a, b)
torch.cuda.synchronize()
print("ok")

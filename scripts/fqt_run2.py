"""Development: K6 register-blocked path only (q = 2^13, d = 1, n_q = 409)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

n = 1 << 16
g = torch.Generator(device="cuda").manual_seed(6)
a = torch.randint(0, 3, (n,), dtype=torch.uint8, device="cuda", generator=g)
b = torch.randint(0, 3, (n,), dtype=torch.uint8, device="cuda", generator=g)
pm = Q.PolymulPlan(3, 1 << 13, 2, 409)
for _ in range(2):
    pm.fqt_mul(a, b)
torch.cuda.synchronize()
print("ok")

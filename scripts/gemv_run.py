"""Development: run the K5 GEMV (8192^2, GF(3^3)) and a 2^26-term fgdp_dot a
few times (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

f = Q.GfqField(3, 3, 1 << 10)
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.randint(0, 27, (8192, 8192), dtype=torch.int32, device="cuda", generator=g)
x = torch.randint(0, 27, (8192,), dtype=torch.int32, device="cuda", generator=g)
v1 = torch.randint(0, 27, (1, 1 << 26), dtype=torch.int32, device="cuda", generator=g)
v2 = torch.randint(0, 27, (1 << 26,), dtype=torch.int32, device="cuda", generator=g)
for _ in range(3):
    f.gemv(A, x)
    f.gemv(v1, v2)
torch.cuda.synchronize()
print("ok")

"""Development: a few launches of one C3 path (for ncu): python scripts/c3_one.py PATH"""
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

path = int(sys.argv[1])
n3 = 1 << 24
a3 = torch.empty(n3 * 3, dtype=torch.uint8, device="cuda")
b3 = torch.empty_like(a3)
Q.gen_pairs(Q.C3.seed, n3, 3, 7, a3, b3)
f3 = Q.GfqField(7, 3, 256)
o3 = torch.empty((n3, 3), dtype=torch.uint8, device="cuda")
for _ in range(4):
    f3.mul_batch(a3, b3, path, out=o3)
torch.cuda.synchronize()
print("ok")

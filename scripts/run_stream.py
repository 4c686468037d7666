"""Run each streaming config once (C1, C2, C3 packed, C3 dlog) for profiling."""
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

which = sys.argv[1:] or ["c1", "c2", "c3p", "c3z"]
if "c2" in which:
    n = 1 << 26
    w = torch.empty(n, dtype=torch.float64, device="cuda")
    Q.gen_words(Q.C2.seed, n, 128, 6, w)
    plan = Q.RedqPlan(5, 128, 6, Q.FLOAT_PREMUL).attach_correction(4)
    out = plan.residues(w)
    plan.sync()
if "c1" in which:
    n1 = 1 << 20
    a1 = torch.empty(n1 * 4, dtype=torch.uint8, device="cuda")
    b1 = torch.empty_like(a1)
    Q.gen_pairs(Q.C1.seed, n1, 4, 3, a1, b1)
    Q.PolymulPlan(3, 32, 4, 1)(a1, b1)
if "c3p" in which or "c3z" in which:
    n3 = 1 << 24
    a3 = torch.empty(n3 * 3, dtype=torch.uint8, device="cuda")
    b3 = torch.empty_like(a3)
    Q.gen_pairs(Q.C3.seed, n3, 3, 7, a3, b3)
    f3 = Q.GfqField(7, 3, 256)
    if "c3p" in which:
        f3.mul_batch(a3, b3, 0)
    if "c3z" in which:
        f3.mul_batch(a3, b3, 1)
torch.cuda.synchronize()
print("ok")

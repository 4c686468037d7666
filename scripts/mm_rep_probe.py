"""Development: device time of the C5 product through the coefficient API
(chunk 64 / 85) and the rep API (reference signature)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

nn, k = 8192, 3
f = Q.GfqField(3, k, 1 << 10)
A = torch.empty(nn * nn * k, dtype=torch.uint8, device="cuda")
B = torch.empty_like(A)
Q.gen_draws(Q.C5.seed, nn * nn * k, 3, A, start=0)
Q.gen_draws(Q.C5.seed, nn * nn * k, 3, B, start=nn * nn * k)
rA = torch.randint(0, 27, (nn, nn), dtype=torch.int32, device="cuda")
rB = torch.randint(0, 27, (nn, nn), dtype=torch.int32, device="cuda")


def t(fn, n=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print("coeff chunk64", t(lambda: f.matmul(A, B, nn, nn, nn, 64)))
print("coeff chunk85", t(lambda: f.matmul(A, B, nn, nn, nn, 85)))
print("coeff chunk0", t(lambda: f.matmul(A, B, nn, nn, nn, 0)))
print("rep", t(lambda: f.matmul_rep(rA, rB)))

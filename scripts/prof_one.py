"""Development: run one headline kernel a few times for an ncu capture
(`ncu -k regex:... -s 2 -c 1`); python scripts/prof_one.py NAME with NAME in
c1 c2 c3p c3d c3l c4 c5 c5f k5g k5d k6"""
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = torch.Generator(device="cuda").manual_seed(1)
if name == "c1":
    n = Q.C1.n
    a = torch.empty(n * 4, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    Q.gen_pairs(Q.C1.seed, n, 4, 3, a, b)
    pm = Q.PolymulPlan(3, 32, 4, 1)
    o = torch.empty((n, 7), dtype=torch.uint8, device="cuda")
    fn = lambda: pm(a, b, out=o)
elif name == "c2":
    n = Q.C2.n
    w = torch.empty(n, dtype=torch.float64, device="cuda")
    Q.gen_words(Q.C2.seed, n, 128, 6, w)
    plan = Q.RedqPlan(5, 128, 6, Q.FLOAT_PREMUL).attach_correction(4)
    o = torch.empty((n, 7), dtype=torch.uint8, device="cuda")
    fn = lambda: plan.residues(w, out=o)
elif name in ("c3p", "c3d", "c3l"):
    n = Q.C3.n
    a = torch.empty(n * 3, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    Q.gen_pairs(Q.C3.seed, n, 3, 7, a, b)
    f = Q.GfqField(7, 3, 256)
    o = torch.empty((n, 3), dtype=torch.uint8, device="cuda")
    path = {"c3p": 0, "c3d": 1, "c3l": 2}[name]
    fn = lambda: f.mul_batch(a, b, path, out=o)
elif name in ("c4", "c5", "c5f"):
    cfg = Q.C4 if name == "c4" else Q.C5
    nn, k = cfg.n, cfg.k
    A = torch.empty(nn * nn * k, dtype=torch.uint8, device="cuda")
    B = torch.empty_like(A)
    Q.gen_draws(cfg.seed, nn * nn * k, 3, A, start=0)
    Q.gen_draws(cfg.seed, nn * nn * k, 3, B, start=nn * nn * k)
    f = Q.GfqField(3, k, cfg.q)
    Cm = torch.empty((nn, nn, k), dtype=torch.uint8, device="cuda")
    rp = "fold" if name == "c5f" else "redq"
    fn = lambda: f.matmul(A, B, nn, nn, nn, cfg.chunk, out=Cm, repack=rp)
elif name in ("k5g", "k5d"):
    f = Q.GfqField(3, 3, 1 << 10)
    if name == "k5g":
        A = torch.randint(0, 27, (8192, 8192), dtype=torch.int32, device="cuda", generator=g)
        x = torch.randint(0, 27, (8192,), dtype=torch.int32, device="cuda", generator=g)
    else:
        A = torch.randint(0, 27, (1, 1 << 26), dtype=torch.int32, device="cuda", generator=g)
        x = torch.randint(0, 27, (1 << 26,), dtype=torch.int32, device="cuda", generator=g)
    fn = lambda: f.gemv(A, x)
elif name == "k6":
    nL = 1 << 20
    a = torch.randint(0, 3, (nL,), dtype=torch.uint8, device="cuda", generator=g)
    b = torch.randint(0, 3, (nL,), dtype=torch.uint8, device="cuda", generator=g)
    o = torch.empty((2 * nL - 1,), dtype=torch.uint8, device="cuda")
    pm = Q.PolymulPlan(3, 1 << 13, 2, 409)
    fn = lambda: pm.fqt_mul(a, b, out=o)
else:
    raise SystemExit(f"unknown kernel {name}")
for _ in range(reps):
    fn()
torch.cuda.synchronize()
print(name, "ok")

"""Quick device timings for development (not the bench contract)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402


def timeit(fn, reps=20, warm=3, flush=None):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[0], ts[len(ts) // 2]


res = {"device": Q.device_info()}
res["dfma_tflops"] = Q.probe_fp64(0, 4096)
res["dmma_tflops"] = Q.probe_fp64(1, 4096)
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
best, med = timeit(lambda: torch.matmul(a, b), reps=5, warm=2)
res["cublas_dgemm_tflops"] = 2 * 8192 ** 3 / (best * 1e-3) / 1e12
del a, b
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

# C2 REDQ
n = 1 << 26
w = torch.empty(n, dtype=torch.float64, device="cuda")
Q.gen_words(Q.C2.seed, n, 128, 6, w)
plan = Q.RedqPlan(5, 128, 6, Q.FLOAT_PREMUL).attach_correction(4)
out = torch.empty((n, 7), dtype=torch.uint8, device="cuda")
best, med = timeit(lambda: plan.residues(w, out=out), flush=flush)
plan.sync()
res["c2_ms"] = [best, med]
res["c2_GBps"] = 15 * n / (best * 1e-3) / 1e9
copy_dst = torch.empty_like(w)
best, med = timeit(lambda: copy_dst.copy_(w), flush=flush)
res["copy_512MB_GBps"] = 2 * 8 * n / (best * 1e-3) / 1e9

# C1
n1 = 1 << 20
a1 = torch.empty(n1 * 4, dtype=torch.uint8, device="cuda")
b1 = torch.empty_like(a1)
Q.gen_pairs(Q.C1.seed, n1, 4, 3, a1, b1)
pm = Q.PolymulPlan(3, 32, 4, 1)
o1 = torch.empty((n1, 7), dtype=torch.uint8, device="cuda")
res["c1_ms_cold"] = timeit(lambda: pm(a1, b1, out=o1), flush=flush)
res["c1_ms_hot"] = timeit(lambda: pm(a1, b1, out=o1))

# C3
n3 = 1 << 24
a3 = torch.empty(n3 * 3, dtype=torch.uint8, device="cuda")
b3 = torch.empty_like(a3)
Q.gen_pairs(Q.C3.seed, n3, 3, 7, a3, b3)
f3 = Q.GfqField(7, 3, 256)
o3 = torch.empty((n3, 3), dtype=torch.uint8, device="cuda")
for path in (0, 1):
    best, med = timeit(lambda: f3.mul_batch(a3, b3, path, out=o3), flush=flush)
    res[f"c3_path{path}_ms"] = [best, med]
    res[f"c3_path{path}_GBps"] = 9 * n3 / (best * 1e-3) / 1e9

# C4 / C5
for cfg in (Q.C4, Q.C5):
    nn, k = cfg.n, cfg.k
    A = torch.empty(nn * nn * k, dtype=torch.uint8, device="cuda")
    B = torch.empty_like(A)
    Q.gen_draws(cfg.seed, nn * nn * k, 3, A, start=0)
    Q.gen_draws(cfg.seed, nn * nn * k, 3, B, start=nn * nn * k)
    f = Q.GfqField(3, k, cfg.q)
    Cm = torch.empty((nn, nn, k), dtype=torch.uint8, device="cuda")
    best, med = timeit(lambda: f.matmul(A, B, nn, nn, nn, cfg.chunk, out=Cm), reps=5, warm=2)
    res[f"c{cfg.cid}_ms"] = [best, med]
    res[f"c{cfg.cid}_tflops"] = 2 * nn ** 3 / (best * 1e-3) / 1e12
print(json.dumps(res, indent=1))

"""One GF(p^k) matmul config on the GPU (profiling / quick timing helper)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cid", type=int, default=5)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--chunk", type=int, default=-1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--repack", default="redq")
a = ap.parse_args()
cfg = Q.CONFIGS[a.cid]
n = a.n or cfg.n
chunk = cfg.chunk if a.chunk < 0 else a.chunk
k = cfg.k
A = torch.empty(n * n * k, dtype=torch.uint8, device="cuda")
B = torch.empty_like(A)
Q.gen_draws(cfg.seed, n * n * k, 3, A, start=0)
Q.gen_draws(cfg.seed, n * n * k, 3, B, start=n * n * k)
f = Q.GfqField(3, k, cfg.q)
Cm = torch.empty((n, n, k), dtype=torch.uint8, device="cuda")
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f.matmul(A, B, n, n, n, chunk, out=Cm, repack=a.repack)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"n={n} k={k} chunk={chunk} repack={a.repack}: {ms:.3f} ms  {2 * n ** 3 / ms / 1e9:.2f} TFLOP/s")

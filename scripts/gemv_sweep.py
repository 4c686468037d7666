"""Development: K5 GEMV / long-dot timings (CUDA graph of 4 launches)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

f = Q.GfqField(3, 3, 1 << 10)
g = torch.Generator(device="cuda").manual_seed(5)
res = {"splits": os.environ.get("QPK_GEMV_SPLITS", "auto")}


def tgraph(fn, n=4, reps=10):
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(n):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / n)
    ts.sort()
    return round(ts[len(ts) // 2] * 1e3, 2)


for m, K in ((8192, 8192), (16384, 16384), (1024, 65536), (65536, 1024)):
    A = torch.randint(0, 27, (m, K), dtype=torch.int32, device="cuda", generator=g)
    x = torch.randint(0, 27, (K,), dtype=torch.int32, device="cuda", generator=g)
    y = torch.empty((m,), dtype=torch.int32, device="cuda")
    us = tgraph(lambda: f.gemv(A, x, out=y))
    res[f"{m}x{K}"] = [us, round(m * K * 4 / us / 1e3, 0)]
    del A
v1 = torch.randint(0, 27, (1, 1 << 26), dtype=torch.int32, device="cuda", generator=g)
v2 = torch.randint(0, 27, (1 << 26,), dtype=torch.int32, device="cuda", generator=g)
y1 = torch.empty((1,), dtype=torch.int32, device="cuda")
us = tgraph(lambda: f.gemv(v1, v2, out=y1), n=2)
res["dot_2^26"] = [us, round((1 << 26) * 8 / us / 1e3, 0)]
print(json.dumps(res))

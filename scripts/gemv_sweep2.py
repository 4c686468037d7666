"""Development: K5 split sweep for few-row shapes (QPK_GEMV_SPLITS per call)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

f = Q.GfqField(3, 3, 1 << 10)
g = torch.Generator(device="cuda").manual_seed(5)


def tgraph(fn, n=3, reps=7):
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
    return round(ts[len(ts) // 2] * 1e3, 1)


for m, K, cands in ((1, 1 << 26, (1480, 2960, 5920, 11840, 23680, 32768)),
                    (128, 1 << 19, (8, 16, 32, 46, 64, 128, 185, 256)),
                    (1024, 65536, (2, 4, 5, 6, 8, 12, 24, 32)),
                    (4096, 16384, (1, 2, 3, 4, 6, 8))):
    A = torch.randint(0, 27, (m, K), dtype=torch.int32, device="cuda", generator=g)
    x = torch.randint(0, 27, (K,), dtype=torch.int32, device="cuda", generator=g)
    y = torch.empty((m,), dtype=torch.int32, device="cuda")
    res = {}
    for c in ("auto",) + cands:
        if c == "auto":
            os.environ.pop("QPK_GEMV_SPLITS", None)
        else:
            os.environ["QPK_GEMV_SPLITS"] = str(c)
        res[c] = tgraph(lambda: f.gemv(A, x, out=y))
    os.environ.pop("QPK_GEMV_SPLITS", None)
    print(json.dumps({"shape": f"{m}x{K}", "us": res}))
    del A

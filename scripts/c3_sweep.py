"""Development: time GF(7^3) elementwise products (C3) for the library named
by QPK_DEV_LIB (or the in-tree build), the way bench.py does: a CUDA graph of
12 launches cycling through 3 buffer sets (453 MB > L2, so every launch reads
and writes HBM); prints one JSON line (per-launch us: best, median)."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

REPS = int(os.environ.get("C3_REPS", "15"))
n3 = 1 << 24
f3 = Q.GfqField(7, 3, 256)
sets = []
for _ in range(3):
    a3 = torch.empty(n3 * 3, dtype=torch.uint8, device="cuda")
    b3 = torch.empty_like(a3)
    Q.gen_pairs(Q.C3.seed, n3, 3, 7, a3, b3)
    sets.append((a3, b3, torch.empty((n3, 3), dtype=torch.uint8, device="cuda")))


def graph_time(path):
    fns = [lambda s=s_: f3.mul_batch(s[0], s[1], path, out=s[2]) for s_ in sets] * 4
    for fn in fns:
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for fn in fns:
            fn()
    ts = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / len(fns))
    ts.sort()
    return ts[0], ts[len(ts) // 2]


res = {"lib": os.path.basename(os.environ.get("QPK_DEV_LIB", "in-tree"))}
for path in (0, 1, 2):
    best, med = graph_time(path)
    res[f"p{path}_us"] = [round(best * 1e3, 2), round(med * 1e3, 2)]
    res[f"p{path}_sha"] = hashlib.sha1(sets[0][2].cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps(res))

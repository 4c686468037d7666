"""Development: per-launch time of the C1 batched polynomial product
(2^20 pairs, k=4, p=3, q=2^5) for the library named by QPK_DEV_LIB."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

n1 = Q.C1.n
pm = Q.PolymulPlan(3, 32, 4, 1)
sets = []
for _ in range(24):
    a = torch.empty(n1 * 4, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    Q.gen_pairs(Q.C1.seed, n1, 4, 3, a, b)
    sets.append((a, b, torch.empty((n1, 7), dtype=torch.uint8, device="cuda")))


def batch(fns, reps=10):
    for fn in fns:
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for fn in fns:
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / len(fns))
    ts.sort()
    return round(ts[len(ts) // 2] * 1e3, 2)


def graph(fns, reps=10):
    for fn in fns:
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for fn in fns:
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / len(fns))
    ts.sort()
    return round(ts[len(ts) // 2] * 1e3, 2)


res = {"lib": os.path.basename(os.environ.get("QPK_DEV_LIB", "in-tree"))}
res["graph_rot_us"] = graph([lambda s=s_: pm(s[0], s[1], out=s[2]) for s_ in sets])
res["graph_hot_us"] = graph([lambda s=sets[0]: pm(s[0], s[1], out=s[2])] * 24)
res["rot_us"] = batch([lambda s=s_: pm(s[0], s[1], out=s[2]) for s_ in sets])
res["hot_us"] = batch([lambda s=sets[0]: pm(s[0], s[1], out=s[2])] * 24)
res["sha"] = hashlib.sha1(sets[0][2].cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps(res))

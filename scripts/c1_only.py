"""Development: C1 polymul at 2^20 pairs, cold (rotating sets) and hot, graph-timed."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

pm = Q.PolymulPlan(3, 32, 4, 1)


def time_graph(fns, reps=20):
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
    return statistics.median(ts)


for lg in (19, 20):
    n = 1 << lg
    sets = []
    for _ in range(24):
        a = torch.empty(n * 4, dtype=torch.uint8, device="cuda")
        b = torch.empty_like(a)
        Q.gen_pairs(7, n, 4, 3, a, b)
        sets.append((a, b, torch.empty((n, 7), dtype=torch.uint8, device="cuda")))
    cold = time_graph([lambda s=s_: pm(s[0], s[1], out=s[2]) for s_ in sets])
    hot = time_graph([lambda s=sets[0]: pm(s[0], s[1], out=s[2])] * 24)
    print(f"n=2^{lg}: cold {cold * 1e3:.2f} us  hot {hot * 1e3:.2f} us")

"""Development: C1 polymul device time per launch vs batch size (graph of
back-to-back launches over rotating sets), to split fixed from per-pair cost."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

pm = Q.PolymulPlan(3, 32, 4, 1)


def time_graph(fns, reps=10):
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


for lg in (12, 14, 16, 18, 19, 20, 21, 22):
    n = 1 << lg
    nsets = max(2, min(48, (400 << 20) // (15 * n)))
    sets = []
    for _ in range(nsets):
        a = torch.empty(n * 4, dtype=torch.uint8, device="cuda")
        b = torch.empty_like(a)
        Q.gen_pairs(7, n, 4, 3, a, b)
        sets.append((a, b, torch.empty((n, 7), dtype=torch.uint8, device="cuda")))
    cold = time_graph([lambda s=s_: pm(s[0], s[1], out=s[2]) for s_ in sets])
    hot = time_graph([lambda s=sets[0]: pm(s[0], s[1], out=s[2])] * nsets)
    print(f"n=2^{lg}: cold {cold * 1e3:.2f} us  hot {hot * 1e3:.2f} us  {15 * n / cold / 1e6:.0f} GB/s cold")
    del sets

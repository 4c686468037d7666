"""Development: launch-latency floor of a C1-sized streaming step (4 MB +
4 MB in, 7 MB out) with torch elementwise kernels and with the C1 kernel, in
CUDA graphs over 24 rotating buffer sets (377 MB > L2), per launch."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

n1 = Q.C1.n


def t(fns, reps=15):
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / len(fns))
    return sorted(ts)[len(ts) // 2] * 1e3


res = {}
sets = [(torch.randint(0, 3, (n1,), dtype=torch.int32, device="cuda"),
         torch.randint(0, 3, (n1,), dtype=torch.int32, device="cuda"),
         torch.empty(n1, dtype=torch.int32, device="cuda")) for _ in range(24)]
res["torch_add_i32_4MBx2_to_4MB_us"] = t([lambda s=s: torch.add(s[0], s[1], out=s[2]) for s in sets])
big = [torch.empty(n1 * 7 // 4 + 1, dtype=torch.int32, device="cuda") for _ in range(24)]
res["torch_fill_7MB_us"] = t([lambda b=b: b.fill_(1) for b in big])
pm = Q.PolymulPlan(3, 32, 4, 1)
sets1 = []
for _ in range(24):
    a1 = torch.empty(n1 * 4, dtype=torch.uint8, device="cuda")
    b1 = torch.empty_like(a1)
    Q.gen_pairs(Q.C1.seed, n1, 4, 3, a1, b1)
    sets1.append((a1, b1, torch.empty((n1, 7), dtype=torch.uint8, device="cuda")))
res["c1_us"] = t([lambda s=s: pm(s[0], s[1], out=s[2]) for s in sets1])
res["c1_hot_us"] = t([lambda s=sets1[0]: pm(s[0], s[1], out=s[2])] * 24)
print(json.dumps(res))

"""Development: time the K5 GEMV (8192^2, GF(3^3)) and the 2^26-term
fgdp_dot for the library named by QPK_DEV_LIB (or the in-tree build);
prints one JSON line (CUDA-event medians, L2 flushed between reps)."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

f = Q.GfqField(3, 3, 1 << 10)
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.randint(0, 27, (8192, 8192), dtype=torch.int32, device="cuda", generator=g)
x = torch.randint(0, 27, (8192,), dtype=torch.int32, device="cuda", generator=g)
v1 = torch.randint(0, 27, (1, 1 << 26), dtype=torch.int32, device="cuda", generator=g)
v2 = torch.randint(0, 27, (1 << 26,), dtype=torch.int32, device="cuda", generator=g)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {"lib": os.path.basename(os.environ.get("QPK_DEV_LIB", "in-tree"))}
for name, fn in (("gemv", lambda: f.gemv(A, x)), ("dot", lambda: f.gemv(v1, v2))):
    for _ in range(3):
        y = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        y = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    res[name + "_us"] = [round(ts[0], 1), round(ts[15], 1)]
    res[name + "_sha"] = hashlib.sha1(y.cpu().numpy().tobytes()).hexdigest()[:10]
print(json.dumps(res))

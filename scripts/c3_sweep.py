"""Development: time GF(7^3) elementwise products (C3) for the library named
by QPK_DEV_LIB (or the in-tree build); prints one JSON line."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402


def timeit(fn, reps=30, warm=3, flush=None):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(BATCH):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / BATCH)
    ts.sort()
    return ts[0], ts[len(ts) // 2]


REPS = int(os.environ.get("C3_REPS", "30"))
BATCH = int(os.environ.get("C3_BATCH", "10"))  # launches per event pair (event clock is ~2 us coarse)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
n3 = 1 << 24
a3 = torch.empty(n3 * 3, dtype=torch.uint8, device="cuda")
b3 = torch.empty_like(a3)
Q.gen_pairs(Q.C3.seed, n3, 3, 7, a3, b3)
f3 = Q.GfqField(7, 3, 256)
o3 = torch.empty((n3, 3), dtype=torch.uint8, device="cuda")
res = {"lib": os.path.basename(os.environ.get("QPK_DEV_LIB", "in-tree"))}
for path in (0, 1, 2):
    o3.zero_()
    best, med = timeit(lambda: f3.mul_batch(a3, b3, path, out=o3), reps=REPS, warm=min(3, REPS), flush=flush)
    res[f"p{path}_us"] = [round(best * 1e3, 2), round(med * 1e3, 2)]
    res[f"p{path}_sha"] = hashlib.sha1(o3.cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps(res))

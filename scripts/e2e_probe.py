"""Development: C2 end-to-end (host buffers through the C-ABI host entry)
time per step; QPK_HOST_CHUNK_LOG2 selects the staging chunk."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402

N = 1 << 26
plan = Q.RedqPlan(5, 128, 6, Q.FLOAT_PREMUL).attach_correction(4)
dw = torch.empty(N, dtype=torch.float64, device="cuda")
Q.gen_words(Q.C2.seed, N, 128, 6, dw)
hw = dw.cpu().pin_memory()
ho = torch.empty((N, 7), dtype=torch.uint8, pin_memory=True)
hw_np, ho_np = hw.numpy(), ho.numpy()
plan.residues(hw_np, out=ho_np)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    plan.residues(hw_np, out=ho_np)
    ts.append(time.perf_counter() - t0)
ts.sort()
print(json.dumps({"chunk_log2": os.environ.get("QPK_HOST_CHUNK_LOG2", "21"), "ms": [round(t * 1e3, 2) for t in ts]}))

"""Development: why the in-process cpu_baseline leg is slower than the
reference arm: time the reference REDQ in a fresh process, after CUDA init,
and after torch CPU ops."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402

stage = sys.argv[1]
if stage in ("cuda", "cpuop"):
    import torch
    torch.cuda.init()
    x = torch.empty(1 << 28, device="cuda")
    if stage == "cpuop":
        y = torch.randn(1 << 24).sum()
        z = x[: 1 << 20].cpu().numpy()
words = bench.c2_words(bench.N_WORDS)
out = np.empty((bench.N_WORDS, 7), np.uint8)
v, kind, cores = bench.c2_reference_rate(words, out, bench.host_threads(), 3, 1)
print(stage, f"{v:.3e}", kind, cores, os.environ.get("OMP_NUM_THREADS"))

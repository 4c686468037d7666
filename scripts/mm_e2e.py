"""Development: C4 / C5 through the host-buffer API (pinned numpy in and out), ms per call."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q  # noqa: E402


def pinned(shape, dtype=torch.uint8):
    return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()


for cid in (4, 5):
    cfg = Q.CONFIGS[cid]
    n, k = cfg.n, cfg.k
    A, B, C = pinned((n, n, k)), pinned((n, n, k)), pinned((n, n, k))
    rng = np.random.default_rng(cid)
    A[:] = rng.integers(0, 3, A.shape)
    B[:] = rng.integers(0, 3, B.shape)
    f = Q.GfqField(3, k, cfg.q)
    f.matmul(A, B, n, n, n, cfg.chunk, out=C)
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        f.matmul(A, B, n, n, n, cfg.chunk, out=C)
    t = (time.perf_counter() - t0) / reps
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    want = f.matmul(dA.view(-1), dB.view(-1), n, n, n, cfg.chunk).cpu().numpy().reshape(n, n, k)
    print(f"C{cid} e2e {t * 1e3:.2f} ms  {2 * n ** 3 / t:.3e} GF ops/s  equal={np.array_equal(C, want)}")

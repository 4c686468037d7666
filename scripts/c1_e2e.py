import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_0710_0510_b200 as Q
n1 = Q.C1.n
pm = Q.PolymulPlan(3, 32, 4, 1)
def pinned(shape): return torch.empty(shape, dtype=torch.uint8, pin_memory=True).numpy()
ha, hb, ho = pinned((n1, 4)), pinned((n1, 4)), pinned((n1, 7))
rng = np.random.default_rng(1)
ha[:] = rng.integers(0, 3, (n1, 4)); hb[:] = rng.integers(0, 3, (n1, 4))
for _ in range(5): pm(ha, hb, out=ho)
t0 = time.perf_counter()
for _ in range(50): pm(ha, hb, out=ho)
t = (time.perf_counter() - t0) / 50
print(f"C1 e2e {t*1e3:.3f} ms/step  {n1/t:.3e} pairs/s")

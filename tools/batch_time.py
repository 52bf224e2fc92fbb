"""Config C timing: python tools/batch_time.py -> kernel window and e2e (median of 20)"""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_19373_b200 as qb  # noqa: E402
from paper_2310_19373_b200 import _lib, instances  # noqa: E402
b = instances.config_batch(4096, 16)
for _ in range(3):
    _lib.solve_batch(b)
ks, es = [], []
for _ in range(20):
    ks.append(_lib.solve_batch(b)[2])
    t0 = time.perf_counter()
    qb.solve_batch(b, as_arrays=True)
    es.append(time.perf_counter() - t0)
print(f"config C kernel window {statistics.median(ks):.4f} ms  e2e {1e3 * statistics.median(es):.4f} ms")

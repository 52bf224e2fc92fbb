"""Config C end to end: the (4096, 16, 16) batch as fp64 and as float32 through solve_batch."""
import os, sys, time, statistics
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_19373_b200 as qb
from paper_2310_19373_b200 import instances
b64 = instances.config_batch(4096, 16)
b32 = b64.astype(np.float32)
for name, b in (("fp64", b64), ("float32", b32)):
    for _ in range(3):
        qb.solve_batch(b, as_arrays=True)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); qb.solve_batch(b, as_arrays=True); ts.append(time.perf_counter() - t0)
    print(f"config C e2e {name}: median {1e3 * statistics.median(ts):.3f} ms, min {1e3 * min(ts):.3f} ms", flush=True)

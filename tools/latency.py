"""Development helper: per-call latency breakdown of small solves (Python API vs C ABI vs kernels)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2310_19373_b200 as qb
from paper_2310_19373_b200 import _lib, instances

for name in sys.argv[1:] or ["A", "B"]:
    c = instances.config_coeffs(name, 0)
    inst = qb.QuboInstance(c)
    for _ in range(20):
        qb.solve_incremental(inst)
    py, cabi, tot, ker, srch = [], [], [], [], []
    for _ in range(200):
        t0 = time.perf_counter()
        qb.solve_incremental(inst)
        py.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        r = _lib.solve(inst.coeffs)
        cabi.append(time.perf_counter() - t0)
        tot.append(r.total_ms * 1e-3)
        ker.append(r.kernel_ms * 1e-3)
        srch.append(r.search_ms * 1e-3)
    t0 = time.perf_counter()
    for _ in range(200):
        qb.QuboInstance(c)
    mk = (time.perf_counter() - t0) / 200
    med = lambda v: 1e6 * float(np.median(v))
    print(f"{name}: n={inst.n} python_api={med(py):.1f}us c_abi_wall={med(cabi):.1f}us c_total={med(tot):.1f}us "
          f"kernels={med(ker):.1f}us search={med(srch):.1f}us launches={r.launches} QuboInstance()={1e6 * mk:.1f}us")

"""Time the table-load coarse kernel against the patched-immediate one (QB_VARIANT_IMM) on a config:
python tools/imm_compare.py [E] [n] [reps]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "E"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = instances.config_coeffs(name, 0, n=n)
_lib.solve(instances.config_coeffs(name, 1, n=n), variant=_lib.VARIANT_COARSE)  # CUDA context, library init
t0 = time.perf_counter()
first = _lib.solve(c, variant=_lib.VARIANT_IMM2)
print(f"first IMM2 call (patch + load + solve): {1e3 * (time.perf_counter() - t0):.2f} ms wall, total_ms {first.total_ms:.2f}, "
      f"module_ms {first.module_ms:.2f}, search {first.search_ms:.3f} ms")
for var, label in ((_lib.VARIANT_COARSE, "coarse"), (_lib.VARIANT_IMM, "imm"), (_lib.VARIANT_IMM2, "imm2")):
    _lib.solve(c, variant=var)
    rs = [_lib.solve(c, variant=var) for _ in range(reps)]
    print(f"{label:7s} search {statistics.median(r.search_ms for r in rs):.3f} ms  kernel {statistics.median(r.kernel_ms for r in rs):.3f} ms"
          f"  total {statistics.median(r.total_ms for r in rs):.3f} ms  argmin {hex(rs[-1].argmin_bits)} value {rs[-1].value!r} variant {rs[-1].variant}")

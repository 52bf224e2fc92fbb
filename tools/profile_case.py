"""Run one config solve twice (warm-up + profiled) for ncu captures: python tools/profile_case.py E [n]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances
name = sys.argv[1] if len(sys.argv) > 1 else "E"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
c = instances.config_coeffs(name, 0, n=n)
for _ in range(2):
    r = _lib.solve(c, variant=variant)
print(name, c.shape[0], r.kernel_ms, hex(r.argmin_bits), r.value)

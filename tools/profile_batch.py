"""Run the config-C batch twice (warm-up + profiled) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances
b = instances.config_batch(4096, 16)
for _ in range(2):
    bits, vals, ms = _lib.solve_batch(b)
print("batch kernel ms", ms)

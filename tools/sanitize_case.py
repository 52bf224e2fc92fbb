"""Small cases touching every kernel, for compute-sanitizer runs (one tool per gpurun call)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2310_19373_b200 as qb
from paper_2310_19373_b200 import _lib, instances

c = instances.config_coeffs("D", 1, n=14)
print("exact", _lib.solve(c).argmin_bits)
c = instances.config_coeffs("E", 1, n=16)
print("float", _lib.solve(c).argmin_bits)
c = instances.config_coeffs("D", 1, n=26)
print("large exact", _lib.solve(c, 0, 0, 2).argmin_bits, _lib.solve(c, 3, 5, 3).argmin_bits)
c = instances.config_coeffs("E", 1, n=27)
print("large float", _lib.solve(c).argmin_bits, _lib.solve(c, variant=_lib.VARIANT_FIELDWALK).argmin_bits)
print("naive", _lib.solve(instances.int_uniform_coeffs(12, 3, -2, 2), 0, 0, 0, _lib.TIE_INTEGER).argmin_bits)
v, xs, cnt = _lib.all_minimisers(np.zeros((12, 12)))
print("all-min", cnt)
b = np.stack([instances.normal_coeffs(10, 50 + i) for i in range(8)])
print("batch", _lib.solve_batch(b)[0][:3])
vals, fields = _lib.prefix_eval(instances.config_coeffs("D", 2, n=22), 12, 0, 64)
print("prefix", vals[:2])
print("sanitize cases done")

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances
c = instances.int_uniform_coeffs(33, 777, -1, 1)
for rnd in range(2):
  for shard in range(3):
    for var in (3, 5, 7, 8, 9, 10):
        r = _lib.solve(c, 0, 0, 0, shard=shard, shard_count=3, variant=var)
        print(rnd, shard, var, r.variant, hex(r.argmin_bits), r.value, hex(r.tie_key), hex(r.value_key), r.prefix_bits, r.search_ms, flush=True)

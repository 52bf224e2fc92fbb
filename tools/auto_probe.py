"""AUTO's kernel choice over repeated solves of one instance: python tools/auto_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances

cases = [("E", 40), ("E", 36), ("E", 32), ("D", 40), ("D", 36), ("D", 32), ("B", 36), ("A", 36)]
for name, n in cases:
    c = instances.config_coeffs(name, 0, n=n)
    ref = _lib.solve(c, variant=_lib.VARIANT_COARSE)
    line = []
    for i in range(4):
        r = _lib.solve(c)
        assert (r.argmin_bits, r.value) == (ref.argmin_bits, ref.value)
        line.append(f"v{r.variant} r{r.retries} {r.search_ms:.3f}ms tot{r.total_ms:.2f} x{r.exact_blocks}")
    print(name, n, " | ".join(line), flush=True)
c = instances.int_uniform_coeffs(36, 777, -1, 1)
ref = _lib.solve(c, variant=_lib.VARIANT_COARSE)
for sh in range(3):
    rs = [_lib.solve(c, shard=sh, shard_count=3) for _ in range(3)]
    print("ties36 shard", sh, " | ".join(f"v{r.variant} r{r.retries} {r.search_ms:.3f}ms x{r.exact_blocks}" for r in rs), flush=True)

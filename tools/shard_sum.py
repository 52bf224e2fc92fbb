"""Search time of the whole space against the sum over S sequential shards (one process, one GPU)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances
c = instances.config_coeffs("E", 0, n=40)
var = _lib.VARIANT_IMM8AS
for S in (1, 2, 4, 8):
    for _ in range(2):
        ts = [_lib.solve(c, shard=s, shard_count=S, variant=var).search_ms for s in range(S)]
    print(S, "shards: sum %.3f ms" % sum(ts), " ".join("%.3f" % t for t in ts), flush=True)

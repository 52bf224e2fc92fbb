"""Development check of the tensor-core variant: same answers as the coarse kernel, search times.
usage: python tools/tc_check.py [configs...]   (E at n = 34..40, D at n = 32..36, B/E float rescaled)"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2310_19373_b200 import _lib, instances

cases = [("E", 34), ("E", 36), ("D", 34), ("E", 38), ("E", 40)]
if len(sys.argv) > 1:
    cases = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]
bad = 0
for name, n in cases:
    c = instances.config_coeffs(name, 0, n=n)
    res = {}
    for var in (_lib.VARIANT_COARSE, _lib.VARIANT_TC):
        r = _lib.solve(c, variant=var)
        ts = []
        for _ in range(3):
            r = _lib.solve(c, variant=var)
            ts.append(r.search_ms)
        res[var] = (r.argmin_bits, r.value, r.variant, float(np.median(ts)), r.prefix_bits, r.exact, r.candidates, r.grid)
    a, b = res[_lib.VARIANT_COARSE], res[_lib.VARIANT_TC]
    ok = a[0] == b[0] and a[1] == b[1]
    bad += not ok
    print(json.dumps(dict(cfg=name, n=n, ok=ok, coarse_ms=a[3], tc_ms=b[3], tc_variant=b[2], k_coarse=a[4], k_tc=b[4],
                          exact=b[5], cand=[a[6], b[6]], argmin=[hex(a[0]), hex(b[0])], value=[a[1], b[1]],
                          grid=[a[7], b[7]], tc_states_per_s=2**n / (b[3] * 1e-3))), flush=True)
print("TC CHECK", "OK" if not bad else f"{bad} MISMATCHES")

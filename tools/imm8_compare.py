"""Byte-packed threshold kernel (QB_VARIANT_IMM8) against the 16-bit patched kernel (QB_VARIANT_IMM):
same answers, search times.  python tools/imm8_compare.py [config] [n,n,...] [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib, instances  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "E"
ns = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [32, 36, 40]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
for n in ns:
    c = instances.config_coeffs(name, 0, n=n)
    out = {}
    for var, label in ((_lib.VARIANT_IMM, "imm"), (_lib.VARIANT_IMM8, "imm8"), (_lib.VARIANT_IMM8S, "imm8s"), (_lib.VARIANT_IMM8A, "imm8a"), (_lib.VARIANT_IMM8AS, "imm8as"), (_lib.VARIANT_IMM8AQ, "imm8aq"), (_lib.VARIANT_BYTE8, "byte8")):
        _lib.solve(c, variant=var)
        rs = [_lib.solve(c, variant=var) for _ in range(reps)]
        r = rs[-1]
        out[label] = (r.argmin_bits, r.value, r.candidates)
        print(f"{name} n={n} {label:5s} search {statistics.median(x.search_ms for x in rs):.3f} ms  kernel "
              f"{statistics.median(x.kernel_ms for x in rs):.3f} ms  total {statistics.median(x.total_ms for x in rs):.3f} ms  "
              f"argmin {hex(r.argmin_bits)} value {r.value!r} cand {r.candidates} variant {r.variant} exact_blocks {r.exact_blocks} of {2 ** (n - 10)}", flush=True)
    print("MATCH" if all(v == out["imm"] for v in out.values()) else f"MISMATCH {out}", flush=True)

"""Timing probe of the ill-conditioned 'one huge term' family (tools/fuzz_common.py family 7): the quantization unit is
set by the 1e9 coefficient, the 1e-3 terms round to zero, so half of all states tie in the quantized value and the
overflow reduction (fp64 re-evaluation of every candidate on the device) does the real work.
python tools/slow_case_probe.py [n] [seed]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_19373_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 34
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
iu = np.triu_indices(n, 1)
c = np.zeros((n, n))
c[iu] = rng.standard_normal(len(iu[0])) * 1e-3
c[0, 0] = -1e9 * rng.random()
for name, var in (("TABLE", _lib.VARIANT_TABLE), ("COARSE", _lib.VARIANT_COARSE), ("IMM8AS", _lib.VARIANT_IMM8AS),
                  ("AUTO", _lib.VARIANT_AUTO), ("AUTO", _lib.VARIANT_AUTO)):
    t0 = time.time()
    r = _lib.solve(c, variant=var)
    print(f"n {n} {name}: {time.time() - t0:.2f} s wall, used {r.variant}, kernel_ms {r.kernel_ms:.1f} search_ms {r.search_ms:.1f} "
          f"collect_ms {r.collect_ms:.1f} candidates {r.candidates} exact_blocks {r.exact_blocks} retries {r.retries} "
          f"argmin {int(r.argmin_bits):#x} value {r.value!r}", flush=True)

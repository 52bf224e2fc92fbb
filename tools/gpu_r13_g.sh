#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "E 32,36,40" "D 32,36,40" "B 32" "A 36"; do set -- $cfg; timeout 600 python tools/imm8_compare.py $1 $2 3 2>&1 | grep -v "^Traceback" ; done | tee gpurun_out/imm8_pass.log
python - <<'PY' 2>&1 | tee -a gpurun_out/imm8_pass.log
import sys; sys.path.insert(0, '.')
from paper_2310_19373_b200 import _lib, instances
for n in (33, 36):
    c = instances.int_uniform_coeffs(n, 777, -1, 1)
    for var in (5, 7, 8, 9, 10):
        _lib.solve(c, variant=var)
        r = _lib.solve(c, variant=var)
        print("ties", n, var, r.search_ms, r.exact_blocks, 2 ** (n - 10), flush=True)
PY

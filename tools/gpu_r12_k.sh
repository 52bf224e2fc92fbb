#!/bin/bash
cd "$(dirname "$0")/.."
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "batch" > gpurun_out/pytest_batch.log 2>&1; echo "batch tests rc $?"; tail -3 gpurun_out/pytest_batch.log
timeout 300 python - <<'PY'
import time, statistics, numpy as np, sys
sys.path.insert(0, '.')
import paper_2310_19373_b200 as qb
from paper_2310_19373_b200 import _lib, instances
b = instances.config_batch(4096, 16)
for _ in range(3): _lib.solve_batch(b)
ks, es = [], []
for _ in range(20):
    ks.append(_lib.solve_batch(b)[2])
    t0 = time.perf_counter(); qb.solve_batch(b, as_arrays=True); es.append(time.perf_counter() - t0)
print("config C kernel window ms", statistics.median(ks), "e2e ms", 1e3 * statistics.median(es))
PY
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:batch_kernel<" -s 4 -c 1 -o gpurun_out/r12_ncu_batch_C2 python tools/profile_batch.py > gpurun_out/ncu_batch2.log 2>&1; echo "ncu rc $?"

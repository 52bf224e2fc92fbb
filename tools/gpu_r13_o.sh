#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests/test_gpu_imm.py -q -x --timeout 900 -k "all_minimisers or gives_up or auto_policy or n34" > gpurun_out/pytest_imm_o.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_imm_o.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2

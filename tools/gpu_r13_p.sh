#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python bench.py --gpus 2 --shared-device --steps 5 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_2rank_shared.json 2> gpurun_out/bench_2rank_shared.err; echo "2-rank rc $?"
tail -3 gpurun_out/bench_2rank_shared.err; head -c 900 gpurun_out/bench_2rank_shared.json
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_2gpu_refused.json 2>&1; echo "2-gpu without flag rc $? (expected nonzero)"; tail -2 gpurun_out/bench_2gpu_refused.json

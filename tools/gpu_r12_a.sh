set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout 1500 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
cat gpurun_out/bench.json

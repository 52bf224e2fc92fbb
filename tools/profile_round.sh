#!/bin/bash
# One GPU call: bench line, ncu launch list of the bench command, ncu --set full of the search kernel.
# usage (under gpurun): tools/profile_round.sh <tag>
tag=${1:-r01}
cd "$(dirname "$0")/.."
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/bench_small_$tag.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch_$tag.log 2>&1
python tools/profile_case.py E > gpurun_out/prof_plain_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:qb::coarse_kernel<" -s 1 -c 1 -o gpurun_out/prof_search_$tag python tools/profile_case.py E \
    > gpurun_out/ncu_full_$tag.log 2>&1
cat gpurun_out/bench_$tag.json

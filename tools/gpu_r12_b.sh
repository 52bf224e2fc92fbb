#!/bin/bash
# round-2 call B: ALU/issue peaks with sampled clocks, bench line, launch list, ncu --set full of the
# search kernel (config E), the table kernel at configs A/B, the batch kernel (config C); a
# compute-sanitizer attempt on the small cases.
cd "$(dirname "$0")/.."
set -x
python tools/alu_peaks.py --out gpurun_out/r12_alu_peaks.json > gpurun_out/alu_peaks.log 2>&1; echo "alu rc $?"
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r12.json 2> gpurun_out/bench_r12.err; echo "bench rc $?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_small.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r12_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch.log 2>&1; echo "launch rc $?"
python tools/profile_case.py E > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:coarse_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_coarse_E python tools/profile_case.py E \
    > gpurun_out/ncu_full_E.log 2>&1; echo "ncu E rc $?"
for cfg in A B; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:table_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_table_$cfg python tools/profile_case.py $cfg \
    > gpurun_out/ncu_full_$cfg.log 2>&1; echo "ncu $cfg rc $?"
done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:batch_kernel<" -s 1 -c 1 -o gpurun_out/r12_ncu_batch_C python tools/profile_batch.py \
  > gpurun_out/ncu_full_C.log 2>&1; echo "ncu C rc $?"
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc $?"
tail -5 gpurun_out/sanitize_memcheck.log
cat gpurun_out/bench_r12.json | cut -c1-1500

#!/bin/bash
# End-of-round evidence: the default bench line (with e2e and cpu_baseline), the other workloads' bench lines,
# then tools/gpu_profile.sh (launch list + ncu --set full).  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "C3 rc=$?"
for cfg in T3 C5 RB; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?"
done
timeout 1200 bash tools/gpu_profile.sh

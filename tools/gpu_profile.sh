#!/bin/bash
# Evidence pass (B200_PROFILING.md recipe): plain run, then the launch list of the same command, then one
# `ncu --set full` capture of the three path kernels on a 16384-image step.  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"polar|radial|cov_|finalize" -c 400 --csv --log-file gpurun_out/launches.csv $CMD \
    > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
CMD2="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --n 16384 --batch 16384"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"polar_kernel|radial_tma|cov_tma" -c 3 \
    -o gpurun_out/prof_full $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"

#!/bin/bash
# Full GPU suite + smoke + default bench line + the RB line (runtime-radix kernel) on the current tree.
cd "$(dirname "$0")/.."
bash tools/gpu_head_check.sh
timeout 900 python bench.py --config RB --no-cpu-baseline --no-e2e > gpurun_out/ev_bench_RB.json 2> gpurun_out/ev_bench_RB.err; echo "RB rc=$?"; cut -c1-400 gpurun_out/ev_bench_RB.json
grep -E "rel l2|eigenvalue" gpurun_out/head_tests.log | tail -40

#!/bin/bash
# W = 5 acceptance: C3 full-size parity (both eps), eps contract, guard bands; then the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_guards.py -m gpu -q -x -s -k "c3 or eps_contract or guard" > gpurun_out/w5_tests.log 2>&1; echo "tests rc=$?"
grep -E "rel l2|eigenvalue|passed|failed|Error|assert" gpurun_out/w5_tests.log | tail -30
timeout 900 python bench.py > gpurun_out/w5_bench_default.json 2> gpurun_out/w5_bench_default.err; echo "bench rc=$?"; cut -c1-900 gpurun_out/w5_bench_default.json

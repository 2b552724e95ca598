#!/bin/bash
# Full GPU suite + smoke + default C3 bench line on the current tree.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/head_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/head_tests.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/head_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/head_smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/head_bench.json 2> gpurun_out/head_bench.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/head_bench.json

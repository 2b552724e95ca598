#!/bin/bash
# Round-2 GPU checks: new parity / collective tests, smoke, one bench line through the 1-rank NCCL path.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-}
timeout 1500 python -m pytest tests/test_gpu_collective.py tests/test_gpu_parity_full.py -m gpu -q -x -s ${K:+-k "$K"} \
    > gpurun_out/r2_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/r2_tests.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke.log
timeout 600 python bench.py --nccl --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_nccl.json 2> gpurun_out/r2_bench_nccl.err
echo "bench rc=$?"; tail -3 gpurun_out/r2_bench_nccl.err; cut -c1-400 gpurun_out/r2_bench_nccl.json

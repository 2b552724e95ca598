#!/bin/bash
# K5 change check: covariance parity / determinism tests, then A/B of the given variant libraries (C3, then C4).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cov or k5 or determinism or spectral or collective" > gpurun_out/k5c_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/k5c_tests.log
bash tools/ab_bench.sh "$@"
CFG=C4 EXTRA="--n 100000" bash tools/ab_bench.sh "$@" 2>&1 | sed 's/^/C4 /'

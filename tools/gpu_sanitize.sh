#!/bin/bash
# One compute-sanitizer tool over tools/sanitize_run.py (small invocations of every kernel family).
# usage: tools/gpu_sanitize.sh memcheck|racecheck|synccheck|initcheck [parts...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TOOL=${1:-memcheck}; shift
python tools/sanitize_run.py "$@" > gpurun_out/san_${TOOL}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/san_${TOOL}_plain.log; exit 1; }
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_run.py "$@" \
    > gpurun_out/san_${TOOL}.log 2>&1
echo "sanitizer $TOOL rc=$?"; tail -4 gpurun_out/san_${TOOL}.log

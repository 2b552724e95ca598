#!/bin/bash
# One ncu --set full capture (with source) of the polar kernel on a 16384-image C3 step.
# usage: tools/prof_polar.sh [tag] [extra bench args]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-polar}
shift
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-default-eps --n 16384 --batch 16384 $*"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"polar_kernel" -s 1 -c 1 \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/${TAG}_ncu.log

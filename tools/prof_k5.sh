#!/bin/bash
# ncu --set full (with source) of the tensor-core K5 on a 65,536-image C3 covariance launch.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python tools/k47_run.py 65536"
timeout 300 $CMD > gpurun_out/k5p_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cov_tma" -s 1 -c 1 -o gpurun_out/k5p $CMD > gpurun_out/k5p_ncu.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/k5p_ncu.log

#!/bin/bash
# ncu --set full of K4 (radial_tma), K5 (cov_tma) and K7 (project) on a 65,536-image C3 run (second pass).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python tools/k47_run.py 65536"
timeout 300 $CMD > gpurun_out/k47_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
  --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed \
  -k regex:"radial_tma|cov_tma|project_kernel" -s 3 -c 3 -o gpurun_out/k47_prof $CMD > gpurun_out/k47_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/k47_ncu.log

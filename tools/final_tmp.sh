#!/bin/bash
cd /root/repo; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/full_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/full_tests.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
bash tools/gpu_evidence.sh

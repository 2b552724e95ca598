#!/bin/bash
# Iteration loop for polar-kernel work: quick parity, bench line, ncu capture of the polar kernel.
# usage: tools/gpu_iter.sh TAG [pytest -k expr]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-iter}
K=${2:-"expand_parity_blobs or eps_contract or expand_parity_large_L or rotation_reflection"}
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-graph > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
python - "$TAG" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_bench.json").read().strip().splitlines()[-1])
print("value %.0f img/s  ms/step %.2f  clocks %s" % (d["value"], d["ms_per_step"], d["clocks"]))
for k, v in d["kernels"].items(): print("  %-14s %8.3f ms" % (k, v["ms_per_step"]))
PY
if [ -z "$NO_NCU" ]; then bash tools/prof_polar.sh ${TAG}_prof; fi

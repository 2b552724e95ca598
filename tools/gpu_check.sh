#!/bin/bash
# One GPU round trip: parity tests (-m gpu) then a short bench; outputs land in gpurun_out/.
# usage: tools/gpu_check.sh [pytest -k expr]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/gpu_tests.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; fi
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print("value %.0f img/s  ms/step %.2f  e2e %s" % (d["value"], d["ms_per_step"], d.get("e2e", {}).get("value")))
    for k, v in d["kernels"].items(): print("  %-14s %8.3f ms  %s" % (k, v["ms_per_step"], v.get("tflops", "")))
except Exception as e: print("no bench line", e)
PY

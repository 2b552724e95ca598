#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_guards.py -m gpu -q -x -s -k "k5_partial or guard or svd_guard or 512_image" > gpurun_out/k5_tests.log 2>&1
echo "tests rc=$?"; grep -E "worst|passed|failed|Error|error" gpurun_out/k5_tests.log | head -20
for cfg in C5 T3; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --no-graph > gpurun_out/k5_bench_$cfg.json 2> gpurun_out/k5_bench_$cfg.err
  echo "$cfg rc=$?"
  python - $cfg <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/k5_bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("%s value %.0f img/s  ms/step %.2f" % (sys.argv[1], d["value"], d["ms_per_step"]), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()})
PY
done

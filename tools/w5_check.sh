#!/bin/bash
# W = 5 (eps = 1e-4) at C3: accuracy probe against the oracle, then A/B bench lines eps 1e-5 / 1e-4 (interleaved).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/w5_probe.py 512 > gpurun_out/w5_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/w5_probe.log | tail -3
for r in 1 2; do for e in 1e-5 1e-4; do
  timeout 600 python bench.py --eps $e --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-default-eps > gpurun_out/w5_bench_${e}_$r.json 2> gpurun_out/w5_bench_${e}_$r.err
  python - $e $r <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/w5_bench_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], "w", d["config"]["w"], "%.0f img/s  ms/step %.3f  polar %.3f" % (d["value"], d["ms_per_step"], d["kernels"]["polar_K1K2K3"]["ms_per_step"]))
except Exception as ex:
    print(sys.argv[1], "failed", ex)
PY
done; done

#!/bin/bash
# A/B of bench.py argument sets on the same box ("--batch 50000" ...), baseline first; two rounds.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
i=0
for r in 1 2; do
  for v in "" "$@"; do
    tag=$(echo "base$v" | tr ' -' '__')
    timeout 600 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-graph $v > gpurun_out/aba_$tag$r.json 2> gpurun_out/aba_$tag$r.err
    python - "$tag$r" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/aba_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print("%-30s %.0f img/s  ms/step %.3f  " % (sys.argv[1], d["value"], d["ms_per_step"]) +
          "  ".join("%s %.3f" % (n[:6], v["ms_per_step"]) for n, v in d["kernels"].items()))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done

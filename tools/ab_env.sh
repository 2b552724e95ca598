#!/bin/bash
# A/B of environment knobs on the same box: baseline, then each "NAME=VALUE[,NAME=VALUE]" argument; two rounds.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-C3}
for r in 1 2; do
  for v in base "$@"; do
    if [ "$v" = base ]; then envs=""; else envs=$(echo "$v" | tr ',' ' '); fi
    tag=$(echo "$v" | tr '=,' '__')
    env $envs timeout 600 python bench.py --config $CFG --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-default-eps > gpurun_out/abe_$tag$r.json 2> gpurun_out/abe_$tag$r.err
    python - "$tag$r" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/abe_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    k = d["kernels"]
    print("%-28s %.0f img/s  ms/step %.3f  " % (sys.argv[1], d["value"], d["ms_per_step"]) +
          "  ".join("%s %.3f" % (n[:6], v["ms_per_step"]) for n, v in k.items()))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done

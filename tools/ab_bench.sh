#!/bin/bash
# A/B of two library builds on the same box: A = lib/libfbspca.so, B = $1 (default lib_alt/libfbspca.so), ABAB.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B=${1:-paper_1412_0781_b200/lib_alt/libfbspca.so}
CFG=${2:-C3}
for r in 1 2; do
  for v in A B; do
    if [ $v = A ]; then unset FBSPCA_LIB; else export FBSPCA_LIB=$PWD/$B; fi
    timeout 600 python bench.py --config $CFG --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ab_$v$r.json 2> gpurun_out/ab_$v$r.err
    python - $v$r <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], "%.0f img/s  ms/step %.3f  polar %.3f" % (d["value"], d["ms_per_step"], d["kernels"]["polar_K1K2K3"]["ms_per_step"]))
PY
  done
done
unset FBSPCA_LIB

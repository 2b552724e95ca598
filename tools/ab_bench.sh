#!/bin/bash
# A/B(/C...) of library builds on the same box: A = lib/libfbspca.so, then each variant directory name given
# (paper_1412_0781_b200/lib_<NAME>/libfbspca.so, built with build.py --lib ... -D ...); two rounds, interleaved.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-C3}
VARS="A $*"
for r in 1 2; do
  for v in $VARS; do
    if [ $v = A ]; then unset FBSPCA_LIB; else export FBSPCA_LIB=$PWD/paper_1412_0781_b200/lib_$v/libfbspca.so; fi
    timeout 600 python bench.py --config $CFG $EXTRA --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-default-eps > gpurun_out/ab_$v$r.json 2> gpurun_out/ab_$v$r.err
    python - $v$r <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], "%.0f img/s  ms/step %.3f  polar %.3f" % (d["value"], d["ms_per_step"], d["kernels"]["polar_K1K2K3"]["ms_per_step"]))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done
unset FBSPCA_LIB

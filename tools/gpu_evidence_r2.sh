#!/bin/bash
# Round-2 evidence: default bench line (C3, with e2e and cpu_baseline), other workloads, K6-K7 timings, the launch
# list of the bench command, then one ncu --set full capture of the polar kernel and of K4 / K5 / K7.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/ev_bench_C3.json 2> gpurun_out/ev_bench_C3.err; echo "C3 rc=$?"
timeout 900 python bench.py --eps 1e-5 --no-cpu-baseline --no-e2e > gpurun_out/ev_bench_C3_eps1e-5.json 2> gpurun_out/ev_bench_C3_eps1e-5.err; echo "C3 eps 1e-5 (w = 6) rc=$?"
for cfg in T3 C5 RB C2; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/ev_bench_$cfg.json 2> gpurun_out/ev_bench_$cfg.err
  echo "$cfg rc=$?"
done
timeout 900 python bench.py --config C4 --n 100000 --no-cpu-baseline --no-e2e > gpurun_out/ev_bench_C4.json 2> gpurun_out/ev_bench_C4.err; echo "C4 rc=$?"
timeout 600 python bench.py --nccl --no-cpu-baseline --no-e2e > gpurun_out/ev_bench_nccl.json 2> gpurun_out/ev_bench_nccl.err; echo "nccl rc=$?"
python tools/time_extras.py > gpurun_out/ev_extras.json 2>&1; echo "extras rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-default-eps"
$CMD > gpurun_out/ev_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"polar|radial|cov_|finalize" -c 400 --csv \
    --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launches.log 2>&1
echo "launches rc=$?"
bash tools/prof_polar.sh ev_polar
bash tools/prof_k47.sh

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 2 1 3 s; do
  SPIC_LANDAU_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v$v.log 2>&1
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_landau_x2 -s 2 -c 1 -o gpurun_out/prof_landau -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log

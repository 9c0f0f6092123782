#!/bin/bash
# ncu --set full on the SiLU ISM kernel (n = 2^20)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python tools/bench_silu.py --reps 2 --sizes 1048576"
timeout 300 $CMD > gpurun_out/silu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_silu -s 4 -c 1 -o gpurun_out/prof_silu -f $CMD > gpurun_out/ncu_silu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_silu.log

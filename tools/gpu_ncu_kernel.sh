#!/bin/bash
# ncu --set full on one kernel of tools/bench_kernels.py: KREGEX (regex), KSKIP (launches to skip)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python tools/bench_kernels.py --reps 3"
timeout 300 $CMD > gpurun_out/plain_k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${KSKIP:-3} -c 1 -o gpurun_out/prof_k -f $CMD > gpurun_out/ncu_k.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k.log

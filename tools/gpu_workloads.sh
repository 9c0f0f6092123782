#!/bin/bash
# bench lines of every workload (no CPU baseline) for profiles/: WLS="c0 c3 ..." to choose
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for W in ${WLS:-c0 c0ss c2ss c2blob c3 c4 c4ss c4blob}; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline > gpurun_out/bench_$W.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$W.log
done

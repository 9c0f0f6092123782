#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/bin_sizes.log
for W in c0 c2 c3; do for V in c r; do
  echo "$W $V" >> gpurun_out/bin_sizes.log
  SPIC_BIN_VARIANT=$V timeout 300 python tools/bench_kernels.py --workload $W --reps 10 >> gpurun_out/bin_sizes.log 2>&1
done; done
echo done >> gpurun_out/bin_sizes.log

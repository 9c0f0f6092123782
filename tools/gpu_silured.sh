#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_silu.py -x -q > gpurun_out/silured_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/silured_tests.log
: > gpurun_out/silured.log
for W in c2 c0; do for V in 1 4; do echo "$W $V" >> gpurun_out/silured.log; SPIC_SILU_REDUCE=$V timeout 300 python tools/bench_kernels.py --workload $W --reps 20 >> gpurun_out/silured.log 2>&1; done; done

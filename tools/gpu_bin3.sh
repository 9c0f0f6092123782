#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "binning or radix or engine_steps or run_matches" > gpurun_out/bin_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bin_tests.log
timeout 600 python tools/hbm_ab.py SPIC_RADIX_STAGED=1 > gpurun_out/bin_ab.log 2>&1; echo "rc=$?" >> gpurun_out/bin_ab.log
for W in c2 c3; do SPIC_BIN_VARIANT=c timeout 300 python tools/bench_kernels.py --workload $W --reps 10 >> gpurun_out/bin_ab.log 2>&1; SPIC_BIN_VARIANT=r timeout 300 python tools/bench_kernels.py --workload $W --reps 10 >> gpurun_out/bin_ab.log 2>&1; done

#!/bin/bash
# Iteration session: GPU tests, bench (packed + scalar pair kernel), ncu --set full on k_landau.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_x2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_x2.log
SPIC_LANDAU_VARIANT=s timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_scalar.log 2>&1; echo "rc=$?" >> gpurun_out/bench_scalar.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
if [ "${NCU:-1}" = "1" ]; then
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_landau -s 2 -c 1 -o gpurun_out/prof_landau -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi

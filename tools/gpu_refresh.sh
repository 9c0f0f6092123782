#!/bin/bash
# Full refresh: GPU tests, smoke, headline bench (c2), c3/c4 bench lines, ncu --set full of the
# HBM kernels (push, deposit) at config-4 size.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c2.log
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3.log
timeout 900 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
for K in k_push k_deposit_bulk_ws k_radix_scatter; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_$K -f python tools/hbm_ab.py > gpurun_out/ncu_$K.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_$K.log
done

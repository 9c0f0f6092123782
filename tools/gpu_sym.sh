#!/bin/bash
# antisymmetric pair path: parity tests + per-op timings (sym 128 / sym 256 / ordered)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "antisym or collision or engine or dist or graph or run_matches" > gpurun_out/sym_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sym_tests.log
for wl in c2ss c3; do
  timeout 300 python tools/bench_kernels.py --workload $wl > gpurun_out/k_${wl}_sym128.json 2>&1
  SPIC_SYM_NT=256 timeout 300 python tools/bench_kernels.py --workload $wl > gpurun_out/k_${wl}_sym256.json 2>&1
  SPIC_LANDAU_VARIANT=o timeout 300 python tools/bench_kernels.py --workload $wl > gpurun_out/k_${wl}_ord.json 2>&1
done

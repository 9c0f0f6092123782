#!/bin/bash
# SiLU / tcgen05 bring-up: self-test first (bounded), then the SiLU parity tests.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_silu.py -x -q -k selftest > gpurun_out/silu_selftest.log 2>&1; echo "rc=$?" >> gpurun_out/silu_selftest.log
timeout 600 python -m pytest tests/test_gpu_silu.py -q > gpurun_out/silu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/silu_tests.log
if [ -n "$SILU_BENCH" ]; then
timeout 600 python tools/bench_silu.py > gpurun_out/silu_bench.log 2>&1; echo "rc=$?" >> gpurun_out/silu_bench.log
fi

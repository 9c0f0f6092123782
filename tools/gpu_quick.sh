#!/bin/bash
# quick loop: GPU tests + default bench (+ optional extra bench args via BENCH_ARGS)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline $BENCH_ARGS > gpurun_out/bench_q.log 2>&1; echo "rc=$?" >> gpurun_out/bench_q.log

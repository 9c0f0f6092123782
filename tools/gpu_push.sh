#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python tools/hbm_ab.py SPIC_PUSH_VARIANT=1/2 > gpurun_out/hbm_ab.log 2>&1; echo "rc=$?" >> gpurun_out/hbm_ab.log

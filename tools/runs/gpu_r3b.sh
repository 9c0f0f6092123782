#!/bin/bash
# SiLU iteration: parity tests of the SiLU kernels, phase trace, launch timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_silu.py -x -q -p no:cacheprovider > gpurun_out/r3b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_tests.log
timeout 120 tools/silu_trace 1048576 > gpurun_out/r3b_trace.log 2>&1
timeout 300 python tools/bench_silu.py --sizes 65536,1048576,16777216 > gpurun_out/r3b_silu_bench.log 2>&1

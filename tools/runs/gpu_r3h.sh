#!/bin/bash
# new kernel-shape parity tests + refreshed full-length runs at the bench sizes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "kernel_shapes" > gpurun_out/r3h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3h_tests.log
timeout 900 python tools/long_run.py --workloads c0,c2,c3 > gpurun_out/r3h_long_runs.jsonl 2> gpurun_out/r3h_long_runs.err; echo "rc=$?" >> gpurun_out/r3h_long_runs.err

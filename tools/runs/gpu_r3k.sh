#!/bin/bash
# step_host with the overlapped x copy: its test + the e2e number of the default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -p no:cacheprovider -k "step_host" > gpurun_out/r3k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3k_tests.log
timeout 900 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/r3k_bench.json 2> gpurun_out/r3k_bench.err

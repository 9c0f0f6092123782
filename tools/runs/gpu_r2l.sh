#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_multirank.py -q -s -p no:cacheprovider > gpurun_out/r2l_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2l_pytest.log
timeout 900 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/r2l_bench_c2.json 2> gpurun_out/r2l_bench_c2.err

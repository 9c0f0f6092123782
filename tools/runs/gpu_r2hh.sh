#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/bench_silu.py --reps 10 --sizes 65536,1048576,16777216 > gpurun_out/r2hh_bench_silu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_silu.py tests/test_gpu_faults.py "tests/test_gpu_parity_at_size.py::test_silu_ism_at_bench_size[c2]" "tests/test_gpu_parity_at_size.py::test_silu_ism_at_bench_size[c3]" -q -s -p no:cacheprovider > gpurun_out/r2hh_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2hh_pytest.log

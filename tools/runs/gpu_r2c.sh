#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/bench_silu.py > gpurun_out/r2c_bench_silu.log 2>&1
timeout 900 python tools/diag_silu_acc.py > gpurun_out/r2c_diag.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q -s -p no:cacheprovider > gpurun_out/r2c_dist.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity_at_size.py tests/test_gpu_silu.py -q -s -p no:cacheprovider > gpurun_out/r2c_size.log 2>&1

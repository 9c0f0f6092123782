#!/bin/bash
# full GPU suite + default bench line + NVTX-filtered ncu launch list of one step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=15 > gpurun_out/r2p_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2p_pytest.log
timeout 1200 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
echo "bench rc=$?" >> gpurun_out/r2p_bench.err
SPIC_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "collide/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p_nvtx_collide.csv python tools/bench_kernels.py --workload c0 --reps 1 > gpurun_out/r2p_nvtx.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2p_nvtx.log

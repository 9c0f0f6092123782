#!/bin/bash
# round-2 re-entry: full gpu suite + the default (config-4) bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2700 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=25 > gpurun_out/r2e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2e_pytest.log
timeout 1200 python bench.py > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
echo "bench rc=$?" >> gpurun_out/r2e_bench.err

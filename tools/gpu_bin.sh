#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "binning or radix or engine_steps or graph_replay or config4_size or run_matches" > gpurun_out/bin_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bin_tests.log
timeout 600 python tools/hbm_ab.py SPIC_RADIX_STAGED=1/2 > gpurun_out/bin_ab.log 2>&1; echo "rc=$?" >> gpurun_out/bin_ab.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bin_launches.csv python tools/bin_micro.py > gpurun_out/bin_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/bin_ncu.log

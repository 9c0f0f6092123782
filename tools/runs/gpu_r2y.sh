#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPIC_RADIX_STAGED=3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "binning or radix or engine_steps or graph_replay or config4_size or run_matches" -p no:cacheprovider > gpurun_out/r2y_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2y_tests.log
timeout 600 python tools/hbm_ab.py SPIC_RADIX_STAGED=2/3 > gpurun_out/r2y_hbm.log 2>&1
SPIC_RADIX_STAGED=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2y_launches.csv python tools/bin_micro.py > gpurun_out/r2y_ncu.log 2>&1

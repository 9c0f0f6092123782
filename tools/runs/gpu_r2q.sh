#!/bin/bash
# DRAM traffic per launch of the dominant kernels at config-4 size (metrics only: few replays)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:k_landau_sym -c 1 --log-file gpurun_out/r2q_landau_c4.csv python tools/sym_sweep.py --workload c4ss --cfgs 0 --reps 1 > gpurun_out/r2q_landau.log 2>&1
echo "rc=$?" >> gpurun_out/r2q_landau.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --kernel-name-base mangled -k regex:k_siluILi1E -c 1 --log-file gpurun_out/r2q_silu_c4.csv python tools/bench_silu.py --reps 1 --sizes 16777216 > gpurun_out/r2q_silu.log 2>&1
echo "rc=$?" >> gpurun_out/r2q_silu.log

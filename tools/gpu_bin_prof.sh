#!/bin/bash
# binning launch list at config-4 size (per-kernel durations)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/bin_micro.py > gpurun_out/bin_micro.log 2>&1; echo "rc=$?" >> gpurun_out/bin_micro.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/bin_launches.csv python tools/bin_micro.py > gpurun_out/bin_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/bin_ncu.log

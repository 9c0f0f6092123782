#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_radix_scatter_b -s 2 -c 2 -o gpurun_out/r2m_scatter python tools/bin_micro.py > gpurun_out/r2m_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2m_ncu.log

#!/bin/bash
# ncu --set full of the shipped antisymmetric pair kernel on the config-4 records
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_landau_sym -c 1 -o gpurun_out/r2aa_landau_sym_c4ss python tools/sym_sweep.py --workload c4ss --cfgs 0 --reps 1 > gpurun_out/r2aa_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2aa_ncu.log

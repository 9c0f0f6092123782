#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/sym_sweep.py --workload c2ss --cfgs 0,9,11,12,13,14 --reps 5 > gpurun_out/r2i_sweep_c2ss.json 2>&1
SPIC_SYM_CFG=9 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_landau_symj -c 1 -o gpurun_out/r2i_symj_c2ss python tools/sym_sweep.py --workload c2ss --cfgs 9 --reps 1 > gpurun_out/r2i_ncu.log 2>&1

#!/bin/bash
# pair kernel: RP = 4 configurations (8 targets per thread) vs the shipped 128 x 4 x 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sym_sweep.py --workload c2ss --cfgs 11,13 > gpurun_out/r3c_c2ss.json 2> gpurun_out/r3c_c2ss.err
timeout 900 python tools/sym_sweep.py --workload c4ss --cfgs 11,13 --reps 3 > gpurun_out/r3c_c4ss.json 2> gpurun_out/r3c_c4ss.err

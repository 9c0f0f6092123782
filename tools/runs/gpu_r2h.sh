#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for wl in c2ss c4ss; do
  timeout 900 python tools/sym_sweep.py --workload $wl --cfgs 0,3 --reps 3 > gpurun_out/r2h_sweep_$wl.json 2>&1
done

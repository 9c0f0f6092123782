#!/bin/bash
cd $GRAFT_REPO_ROOT
for wl in c2ss c4ss; do
  timeout 600 python tools/sym_sweep.py --workload $wl --cfgs 0,5,6,7,8 --reps 3 > gpurun_out/r2d_sweep_$wl.json 2>&1
done

#!/bin/bash
# j-split sweep of the new default pair-kernel shape at configs 0, 2, 3, 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for wl in c0ss c2ss c3 c4ss; do
  timeout 900 python tools/split_sweep.py $wl > gpurun_out/r3e_split_$wl.json 2> gpurun_out/r3e_split_$wl.err
done

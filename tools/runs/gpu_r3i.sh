#!/bin/bash
# the decomposed (multi-GPU) bench path at one rank with the final kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPIC_FORCE_DIST=1 timeout 900 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/r3i_bench_c2_forcedist.json 2> gpurun_out/r3i_bench_c2_forcedist.err
SPIC_FORCE_DIST=1 timeout 1200 python bench.py --workload c4 --no-cpu-baseline --no-e2e > gpurun_out/r3i_bench_c4_forcedist.json 2> gpurun_out/r3i_bench_c4_forcedist.err

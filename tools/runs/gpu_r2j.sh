#!/bin/bash
# round-2 bench lines: default (c4) line, c2/c3 lines, forced-decomposition one-rank lines, c4ss reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r2j_bench_c4.json 2> gpurun_out/r2j_bench_c4.err
timeout 900 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/r2j_bench_c2.json 2> gpurun_out/r2j_bench_c2.err
SPIC_FORCE_DIST=1 timeout 900 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/r2j_bench_c2_forcedist.json 2> gpurun_out/r2j_bench_c2_forcedist.err
SPIC_FORCE_DIST=1 timeout 1200 python bench.py --workload c4 --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_c4_forcedist.json 2> gpurun_out/r2j_bench_c4_forcedist.err
timeout 900 python bench.py --impl reference --workload c4ss --steps 2 --warmup 1 > gpurun_out/r2j_ref_c4ss.json 2> gpurun_out/r2j_ref_c4ss.err
timeout 900 python bench.py --impl reference --workload c4 --steps 2 --warmup 1 > gpurun_out/r2j_ref_c4.json 2> gpurun_out/r2j_ref_c4.err

#!/bin/bash
# default bench line + reference arm + config 2 with the final kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r3n_bench.json 2> gpurun_out/r3n_bench.err; echo "rc=$?" >> gpurun_out/r3n_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r3n_ref.json 2> gpurun_out/r3n_ref.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/r3n_bench_c2.json 2> gpurun_out/r3n_bench_c2.err

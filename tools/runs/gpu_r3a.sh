#!/bin/bash
# SiLU ISM phase trace (CTA 0) + per-size launch timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 tools/silu_trace 1048576 > gpurun_out/r3a_trace.log 2>&1
timeout 120 tools/silu_trace_g3 1048576 > gpurun_out/r3a_trace_g3.log 2>&1
timeout 300 python tools/bench_silu.py --sizes 1048576,16777216 > gpurun_out/r3a_silu_bench.log 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 tools/silu_trace 1048576 > gpurun_out/r3l_trace.log 2>&1

#!/bin/bash
# coalesced accumulator-window layout: SiLU tests incl. the at-size ones (flushes), trace, timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_silu.py -x -q -p no:cacheprovider > gpurun_out/r3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.log
timeout 900 python -m pytest tests/test_gpu_parity_at_size.py -x -q -p no:cacheprovider -k "silu and (c2 or c3)" > gpurun_out/r3m_tests_size.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests_size.log
timeout 120 tools/silu_trace 1048576 > gpurun_out/r3m_trace.log 2>&1
timeout 300 python tools/bench_silu.py --sizes 65536,1048576,16777216 > gpurun_out/r3m_silu_bench.log 2>&1

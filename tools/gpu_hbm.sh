#!/bin/bash
# push/deposit A/B: parity tests of the variants + the config-4-size HBM microbench per variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "deposit_variants or push_matches or pic_matches or engine_steps or graph_replay or dist_engine or unfused or vml_engine" > gpurun_out/hbm_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hbm_tests.log
timeout 900 python tools/hbm_ab.py SPIC_PUSH_VARIANT=1/2 > gpurun_out/hbm_ab.log 2>&1; echo "rc=$?" >> gpurun_out/hbm_ab.log

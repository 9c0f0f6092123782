#!/bin/bash
# push/deposit A/B: parity tests of the variants + the config-4-size HBM microbench per variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "deposit_variants or push_matches or pic_matches or engine_steps or graph_replay or dist_engine or unfused or vml_engine" > gpurun_out/hbm_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hbm_tests.log
timeout 900 python tools/hbm_ab.py SPIC_DEP_VARIANT=4/5 > gpurun_out/hbm_ab.log 2>&1; SPIC_DEP_VARIANT=5 timeout 900 python tools/hbm_ab.py SPIC_DEP_CFG=1024,3,4/1024,4,3/2048,2,4/1024,2,7/1024,3,3/768,3,5 >> gpurun_out/hbm_ab.log 2>&1; echo "rc=$?" >> gpurun_out/hbm_ab.log

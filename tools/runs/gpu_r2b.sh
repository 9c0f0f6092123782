#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python tools/diag_silu_acc.py > gpurun_out/r2b_diag.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity_at_size.py -k "config0_100" -x -q -s -p no:cacheprovider > gpurun_out/r2b_c0100.log 2>&1

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "homogeneous or antisymmetric or collision or pair_paths or engine_steps or dist_engine" > gpurun_out/c1_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c1_tests.log
timeout 600 python -c "
import json, torch, bench
from paper_2603_25832_b200 import _lib
_lib.load(build_if_missing=False)
dev = torch.device('cuda', 0)
peak = bench.measure_fp32_peak(torch, dev) if hasattr(bench, 'measure_fp32_peak') else None
for _ in range(2):
    print(json.dumps(bench.config1_microbench(torch, dev)))
" > gpurun_out/c1.log 2>&1; echo "rc=$?" >> gpurun_out/c1.log

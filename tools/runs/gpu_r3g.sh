#!/bin/bash
# M <= 2 (minimum-image) pair kernel shape A/B on the config-1 microbench + its parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 0 11; do
SPIC_SYM_CFG=$c timeout 300 python - > gpurun_out/r3g_c1_$c.json 2> gpurun_out/r3g_c1_$c.err <<'PY'
import json, torch, bench
from paper_2603_25832_b200 import _lib
_lib.load(build_if_missing=False)
print(json.dumps(bench.config1_microbench(torch, torch.device("cuda", 0))))
PY
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_units.py tests/test_gpu_acceptance.py -x -q -p no:cacheprovider -k "collision or landau or minimum or M1 or M2 or image or config1 or stencil or A1 or conservation or antisym" > gpurun_out/r3g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_tests.log
timeout 600 python -m pytest tests/test_gpu_parity_at_size.py -x -q -p no:cacheprovider -k "config1" > gpurun_out/r3g_tests_size.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_tests_size.log

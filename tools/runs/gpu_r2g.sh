#!/bin/bash
# pair kernel: fused negation (fnms2) A/B + G=4 configurations; pair-kernel parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for wl in c2ss c4ss; do
  timeout 900 python tools/sym_sweep.py --workload $wl --cfgs 0,6,7 --reps 3 > gpurun_out/r2g_sweep_$wl.json 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_at_size.py -k "landau or collision or pair or antisym or config1 or config0_100" -q -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2g_pytest.log

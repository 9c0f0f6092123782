#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for wl in c2ss c4ss; do
  timeout 900 python tools/sym_sweep.py --workload $wl --cfgs 0 --reps 3 > gpurun_out/r2ff_sweep_$wl.json 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_units.py tests/test_gpu_acceptance.py tests/test_gpu_dist.py tests/test_gpu_faults.py -q -p no:cacheprovider > gpurun_out/r2ff_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2ff_pytest.log
timeout 1500 python -m pytest tests/test_gpu_parity_at_size.py -q -s -p no:cacheprovider -k "collision or config1 or config0_100 or weibel or dv2 or blob_50" > gpurun_out/r2ff_size.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2ff_size.log

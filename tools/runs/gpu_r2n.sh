#!/bin/bash
# shared-space addressing of the dynamic smem bases (no generic LD/ST), column-scan of radix counts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for wl in c2ss c4ss; do
  timeout 900 python tools/sym_sweep.py --workload $wl --cfgs 0 --reps 3 > gpurun_out/r2n_sweep_$wl.json 2>&1
done
timeout 600 python tools/hbm_ab.py SPIC_RADIX_STAGED=2 > gpurun_out/r2n_hbm.log 2>&1
timeout 900 python tools/bench_kernels.py > gpurun_out/r2n_kernels.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/r2n_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2n_pytest.log

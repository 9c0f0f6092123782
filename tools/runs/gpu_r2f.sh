#!/bin/bash
# fault-path / score_test parity, the partial-range fix, pair-kernel config sweep, ncu of the shipped pair kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_faults.py "tests/test_gpu_parity.py::test_antisymmetric_pair_path_partial_cell_range" tests/test_gpu_parity.py -q -s -p no:cacheprovider > gpurun_out/r2f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f_pytest.log
for wl in c2ss c4ss; do
  timeout 900 python tools/sym_sweep.py --workload $wl --cfgs 0,5,9,10 --reps 3 > gpurun_out/r2f_sweep_$wl.json 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_landau_sym -c 1 -o gpurun_out/r2f_landau_sym_c2ss python tools/sym_sweep.py --workload c2ss --cfgs 0 --reps 1 > gpurun_out/r2f_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2f_ncu.log

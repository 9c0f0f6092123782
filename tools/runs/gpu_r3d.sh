#!/bin/bash
# new default pair-kernel shape (64 x 10 targets): parity tests, blob-kernel shape A/B, c4 line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_acceptance.py tests/test_gpu_reference_units.py -x -q -p no:cacheprovider > gpurun_out/r3d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_tests.log
timeout 900 python -m pytest tests/test_gpu_parity_at_size.py -x -q -p no:cacheprovider -k "collision or config1" > gpurun_out/r3d_tests_size.log 2>&1; echo "rc=$?" >> gpurun_out/r3d_tests_size.log
for c in 0 1 2; do
  SPIC_BLOB_SYM_CFG=$c timeout 600 python bench.py --workload c2blob --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/r3d_c2blob_$c.json 2> gpurun_out/r3d_c2blob_$c.err
  SPIC_BLOB_SYM_CFG=$c timeout 600 python bench.py --workload c4blob --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/r3d_c4blob_$c.json 2> gpurun_out/r3d_c4blob_$c.err
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3d_bench_c4.json 2> gpurun_out/r3d_bench_c4.err

#!/bin/bash
# antisymmetric pair path: full GPU suite, default bench, launch list, ncu of k_landau_sym
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --workload c2ss --no-cpu-baseline > gpurun_out/bench_c2ss.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
CMD="python tools/bench_kernels.py --workload c2ss --reps 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_landau_sym -s 3 -c 1 -o gpurun_out/prof_sym -f $CMD > gpurun_out/ncu_k.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k.log

#!/bin/bash
# Round evidence: GPU tests, smoke, bench (N=1) + reference arms for every workload, launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c2.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_c2_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_c2_ref.log
for wl in c2ss c0 c0ss c3 c4 c4ss c2blob c4blob; do
  timeout 900 python bench.py --workload $wl > gpurun_out/bench_$wl.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$wl.log
done
timeout 900 python bench.py --workload c3 --impl reference > gpurun_out/bench_c3_ref.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log

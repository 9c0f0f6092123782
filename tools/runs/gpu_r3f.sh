#!/bin/bash
# round-2 late verification: smoke, whole GPU suite, default bench + reference arm, ncu captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r3f_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r3f_smoke.log
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/r3f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3f_pytest.log
timeout 1200 python bench.py > gpurun_out/r3f_bench.json 2> gpurun_out/r3f_bench.err
echo "bench rc=$?" >> gpurun_out/r3f_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r3f_ref.json 2> gpurun_out/r3f_ref.err
echo "ref rc=$?" >> gpurun_out/r3f_ref.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/r3f_bench_c2.json 2> gpurun_out/r3f_bench_c2.err
# ncu --set full: SiLU ISM kernel at n = 2^20, pair kernel on the config-4 records
CMD="python tools/bench_silu.py --reps 2 --sizes 1048576"
timeout 300 $CMD > gpurun_out/r3f_silu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_silu -s 4 -c 1 -o gpurun_out/r3f_prof_silu -f $CMD > gpurun_out/r3f_ncu_silu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r3f_ncu_silu.log
CMD="python tools/bench_kernels.py --reps 2 --workload c4ss"
timeout 600 $CMD > gpurun_out/r3f_k_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_landau_sym -s 2 -c 1 -o gpurun_out/r3f_prof_pair -f $CMD > gpurun_out/r3f_ncu_pair.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r3f_ncu_pair.log
# launch list of the default bench command
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/r3f_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/r3f_launches.csv $CMD > gpurun_out/r3f_ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r3f_ncu_launch.log

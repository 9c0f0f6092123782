#!/bin/bash
# round-2 final verification: smoke, the whole GPU suite, the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2x_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2x_smoke.log
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/r2x_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2x_pytest.log
timeout 1200 python bench.py > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err
echo "bench rc=$?" >> gpurun_out/r2x_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2x_ref.json 2> gpurun_out/r2x_ref.err
echo "ref rc=$?" >> gpurun_out/r2x_ref.err

#!/bin/bash
# same-box A/B of two builds of the library (tools/ab/lib_old.so, lib_new.so): SiLU timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/r3o_ab.log
for rep in 1 2 3; do
for v in new old; do
  cp tools/ab/lib_$v.so paper_2603_25832_b200/lib/libscorepic_b200.so
  echo "== $v $rep" >> gpurun_out/r3o_ab.log
  timeout 300 python tools/bench_silu.py --sizes 1048576,16777216 2>&1 | cut -c1-110 >> gpurun_out/r3o_ab.log
done
done
cp tools/ab/lib_new.so paper_2603_25832_b200/lib/libscorepic_b200.so

#!/bin/bash
# A/B the sweep kernels of several libptmh builds on one GPU (run under gpurun):
#   tools/ab_libs.sh "base prep cg" "c3 1024,32 c4" [rounds]
# variants/libptmh_<name>.so ("cur" = the in-tree build); tools/time_sweep.py timings.
names=$1; shapes=$2; rounds=${3:-2}
for r in $(seq $rounds); do
  for n in $names; do
    if [ "$n" = cur ]; then lib=$PWD/paper_2512_03825_b200/libptmh.so; else lib=$PWD/variants/libptmh_$n.so; fi
    PTMH_LIB=$lib python tools/time_sweep.py $shapes 2>&1 | sed "s/^/$n: /"
  done
done

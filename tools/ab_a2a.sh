#!/bin/bash
# A/B of experiment builds on the config-2 alltoallv bench (run on a GPU box).
# usage: tools/ab_a2a.sh N "topo ..." lib1.so lib2.so ...   ("default" = in-tree build)
N=$1; topos=$2; shift 2
for l in "$@"; do
  if [ "$l" = default ]; then unset FASTB200_LIB; else export FASTB200_LIB=$l; fi
  for t in $topos; do echo -n "$l "; bash tools/sweep_a2a.sh $N "128 1048576 $t"; done
done

#!/bin/bash
# A/B of variant builds (exp/<name>/libtrioalign_b200.so) on one box:
# usage: tools/gpu_ab.sh "<ab_quick args>" name1 name2 ...  (in-tree build = "tree")
mkdir -p gpurun_out
ARGS=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = tree ]; then timeout 600 python tools/ab_quick.py $ARGS; else TA_LIB_PATH_EXPERIMENT=exp/$v/libtrioalign_b200.so timeout 600 python tools/ab_quick.py $ARGS; fi
  done
done

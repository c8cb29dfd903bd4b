#!/bin/bash
# same-box A/B of library variants: scripts/ab_libs.sh "cfg4 cfg3" default nu1 nu4 ...
cfgs=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    for c in $cfgs; do
      if [ "$lib" = default ]; then L=""; else L=$PWD/paper_1909_05098_b200/libfedheat_b200_$lib.so; fi
      FH_LIB=$L timeout 300 python scripts/sweep.py --config $c --parts 0 --modes -1 --stages 2 --steps 100 2>&1 | grep part_nodes | sed "s/^/$lib $c rep$rep /"
    done
  done
done

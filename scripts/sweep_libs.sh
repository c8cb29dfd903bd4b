#!/bin/bash
# Time the default cfg4 step with each variant library given on the command line.
for v in "$@"; do
  lib=paper_1909_05098_b200/libfedheat_b200_$v.so; [ "$v" = base ] && lib=paper_1909_05098_b200/libfedheat_b200.so
  echo "== $v"; FH_LIB=$PWD/$lib timeout 300 python scripts/sweep.py --parts 1536 --modes 5 --stages 2 --steps 100 ${SWEEP_ARGS} 2>&1 | grep part_nodes
done

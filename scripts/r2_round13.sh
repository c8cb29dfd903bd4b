#!/bin/bash
# compile-time knobs re-measured on the final kernels: vector zeroing of the accumulators, halo gather unroll 4, node-loop unroll 1 / 4
out=gpurun_out/r13; mkdir -p $out
sw() { timeout 600 python scripts/sweep.py --modes -1 --stages 2 --steps 100 --bench-layout "$@" 2>&1 | grep "part_nodes\|Error\|error" ; }
for rep in 1 2; do
  for lib in default vz su4 nu1 nu4; do
    if [ $lib = default ]; then L=""; else L=$PWD/paper_1909_05098_b200/libfedheat_b200_$lib.so; fi
    for c in "cfg4 32" "cfg3 32"; do set -- $c; FH_LIB=$L sw --config $1 --precision $2 --parts 0 | sed "s/^/$lib $1 f$2 rep$rep /"; done
  done
done | tee $out/ab.jsonl

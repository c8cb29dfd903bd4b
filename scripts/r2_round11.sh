#!/bin/bash
# rolling L2 prefetch of the batch records ahead of the TMA ring (FH_LEAN_PF = 2, 4) against the default library
out=gpurun_out/r11; mkdir -p $out
sw() { timeout 600 python scripts/sweep.py --modes -1 --stages 2 --steps 100 --bench-layout "$@" 2>&1 | grep "part_nodes\|Error\|error" ; }
for rep in 1 2; do
  for lib in default pf2 pf4; do
    if [ $lib = default ]; then L=""; else L=$PWD/paper_1909_05098_b200/libfedheat_b200_$lib.so; fi
    for c in "cfg3 32" "cfg3 64" "cfg4 32"; do set -- $c; FH_LIB=$L sw --config $1 --precision $2 --parts 0 | sed "s/^/$lib $1 f$2 rep$rep /"; done
  done
done | tee $out/ab.jsonl

#!/bin/bash
# ring depth re-measured with the smaller T-only tiles
out=gpurun_out/r8; mkdir -p $out
sw() { timeout 600 python scripts/sweep.py --modes -1 --steps 100 --bench-layout "$@" 2>&1 | grep "part_nodes\|Error\|error" ; }
for c in "cfg3 32" "cfg3 64" "cfg4 32"; do set -- $c; sw --config $1 --precision $2 --parts 0 --stages 2,3 | sed "s/^/$1 f$2 /"; done | tee $out/stages.jsonl

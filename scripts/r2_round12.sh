#!/bin/bash
# cfg5: one LEAN 3 launch for every material-0 tile (kind_split = 1) against the split launches
out=gpurun_out/r12; mkdir -p $out
sw() { timeout 600 python scripts/sweep.py --modes -1 --stages 2 --steps 100 --bench-layout "$@" 2>&1 | grep "part_nodes\|Error\|error" ; }
for rep in 1 2 3; do
  sw --config cfg5 --precision 32 --parts 0 | sed "s/^/split rep$rep /"
  sw --config cfg5 --precision 32 --parts 0 --tuning kind_split=1 | sed "s/^/one-launch rep$rep /"
done | tee $out/ab.jsonl

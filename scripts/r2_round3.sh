#!/bin/bash
# new defaults (5 hex / 6 tet CTAs per SM), tet accumulator rows for fp64, then stamped resident kernel
out=gpurun_out/r3; mkdir -p $out
sw() { timeout 600 python scripts/sweep.py --modes -1 --stages 2 --steps 100 --bench-layout "$@" 2>&1 | grep "part_nodes\|Error\|error" ; }
for c in "cfg4 32" "cfg3 32" "cfg3 64" "cfg5 32"; do set -- $c; sw --config $1 --precision $2 --parts 0 | sed "s/^/default $1 f$2 /"; done | tee $out/defaults.jsonl
for r in 2 3; do sw --config cfg3 --precision 64 --parts 0,512 --tuning tet_rows=$r | sed "s/^/rows$r cfg3 f64 /"; done | tee $out/rows_f64.jsonl
sw --config cfg3 --precision 32 --parts 0 --tuning tet_rows=3 | sed "s/^/rows3 cfg3 f32 /" | tee $out/rows_f32.jsonl
bash scripts/r2_stamped.sh

#!/bin/bash
# tet tile size x accumulator rows (one- and two-wave launches), then ncu captures of the new kernels
out=gpurun_out/r4; mkdir -p $out
sw() { timeout 600 python scripts/sweep.py --modes -1 --stages 2 --steps 100 --bench-layout "$@" 2>&1 | grep "part_nodes\|Error\|error" ; }
for r in 2 3 4; do sw --config cfg3 --precision 32 --parts 0,1170,871 --tuning tet_rows=$r | sed "s/^/rows$r cfg3 f32 /"; done | tee $out/tet_f32.jsonl
for r in 2 3; do sw --config cfg3 --precision 64 --parts 0,871,700 --tuning tet_rows=$r | sed "s/^/rows$r cfg3 f64 /"; done | tee $out/tet_f64.jsonl

#!/bin/bash
# same-box A/B: the library at an older commit (worktree _old/) vs the current one
mkdir -p gpurun_out/abold
for rep in 1 2; do
  for c in cfg3 cfg5 cfg4; do
    (cd _old && timeout 300 python scripts/sweep.py --config $c --parts 0 --modes 5 --stages 2 --steps 100 2>&1 | grep part_nodes | sed "s/^/old $c /")
    timeout 300 python scripts/sweep.py --config $c --parts 0 --modes 5 --stages 2 --steps 100 2>&1 | grep part_nodes | sed "s/^/new $c /"
  done
done

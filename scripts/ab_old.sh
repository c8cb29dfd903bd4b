#!/bin/bash
# Same-box A/B of the step kernel: an older commit checked out as a worktree in
# _old/ (git worktree add _old <commit>; make -C _old/paper_1909_05098_b200/csrc)
# against the current tree, default tile sizes, each config twice:
#   bash scripts/ab_old.sh [configs...]   (default cfg3 cfg5 cfg4)
mkdir -p gpurun_out/abold
cfgs="${@:-cfg3 cfg5 cfg4}"
for rep in 1 2; do
  for c in $cfgs; do
    (cd _old && timeout 300 python scripts/sweep.py --config $c --parts 0 --modes 5 --stages 2 --steps 100 2>&1 | grep part_nodes | sed "s/^/old $c /")
    timeout 300 python scripts/sweep.py --config $c --parts 0 --modes 5 --stages 2 --steps 100 2>&1 | grep part_nodes | sed "s/^/new $c /"
  done
done

#!/bin/bash
# ncu --set full capture of one step-kernel launch for each config given: scripts/profile_cfg.sh cfg3 cfg5
out=gpurun_out/prof; mkdir -p $out
for c in "$@"; do
  cmd="python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
  $cmd > $out/plain_$c.log 2>&1 || { echo "$c plain run failed"; continue; }
  ncu --set full --clock-control none --import-source on -k regex:k_tiled_step -s ${NCU_SKIP:-5} -c ${NCU_COUNT:-1} -o $out/tiled_$c $cmd > $out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done

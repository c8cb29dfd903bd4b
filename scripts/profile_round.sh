#!/bin/bash
# Round profile artifacts (one GPU): plain bench, ncu launch list, ncu full capture of the step kernel.
out=gpurun_out/prof; mkdir -p $out
cmd="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
$cmd > $out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_tiled_step -s 5 -c 1 -o $out/tiled_cfg4 $cmd > $out/ncu_full.log 2>&1; echo "full rc=$?"

#!/bin/bash
# Round profile artifacts (one GPU): ncu launch list of the default bench and
# ncu --set full captures of the step kernel on cfg4 and cfg3.
out=gpurun_out/prof; mkdir -p $out
cmd="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
$cmd > $out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_tiled_step -s 5 -c 1 -o $out/tiled_cfg4 $cmd > $out/ncu_full.log 2>&1; echo "full cfg4 rc=$?"
cmd3="python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
$cmd3 > $out/plain3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_tiled_step -s 5 -c 1 -o $out/tiled_cfg3 $cmd3 > $out/ncu_full3.log 2>&1; echo "full cfg3 rc=$?"

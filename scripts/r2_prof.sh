#!/bin/bash
# ncu --set full of the step-kernel launches of one step: scripts/r2_prof.sh CONFIG PRECISION [LAUNCHES_PER_STEP]
out=gpurun_out/prof2; mkdir -p $out
c=$1; p=$2; n=${3:-1}
cmd="python bench.py --config $c --precision $p --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
$cmd > $out/plain_${c}_f$p.log 2>&1 || { echo "plain $c $p failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled_step -s $((5 * n)) -c $n -o $out/tiled_${c}_f$p $cmd > $out/ncu_${c}_f$p.log 2>&1; echo "ncu $c f$p rc=$?"

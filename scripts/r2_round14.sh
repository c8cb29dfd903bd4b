#!/bin/bash
# cfg5: side stream (mixed / general tiles) at the highest stream priority, against default priority; bench.py and sweep.py
out=gpurun_out/r14; mkdir -p $out
PREV=$PWD/paper_1909_05098_b200/libfedheat_b200_prev.so
for rep in 1 2 3; do
  for lib in prev new; do
    if [ $lib = prev ]; then L=$PREV; else L=""; fi
    FH_LIB=$L timeout 600 python bench.py --config cfg5 --steps 100 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib bench rep$rep', round(d['ms_per_step'],4))"
  done
done | tee $out/ab.txt
for lib in prev new; do
  if [ $lib = prev ]; then L=$PREV; else L=""; fi
  FH_LIB=$L timeout 600 python scripts/sweep.py --config cfg5 --precision 32 --parts 0 --modes -1 --stages 2 --steps 100 --bench-layout 2>&1 | grep part_nodes | sed "s/^/$lib sweep /"
done | tee -a $out/ab.txt

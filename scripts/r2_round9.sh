#!/bin/bash
# trash-slot accumulation in the LEAN loops: parity subset, A/B against the previous library; ring depth sweep
out=gpurun_out/r9; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_extensions.py tests/test_gpu_robustness.py tests/test_gpu_dist.py tests/test_gpu_dist_host.py -m gpu -x -q > $out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -5 $out/pytest_quick.log
sw() { timeout 600 python scripts/sweep.py --modes -1 --stages 2 --steps 100 --bench-layout "$@" 2>&1 | grep "part_nodes\|Error\|error" ; }
PREV=$PWD/paper_1909_05098_b200/libfedheat_b200_prev.so
for rep in 1 2; do
  for lib in prev new; do
    if [ $lib = prev ]; then L=$PREV; else L=""; fi
    for c in "cfg4 32" "cfg3 32" "cfg3 64" "cfg5 32"; do set -- $c; FH_LIB=$L sw --config $1 --precision $2 --parts 0 | sed "s/^/$lib $1 f$2 rep$rep /"; done
  done
done | tee $out/ab.jsonl
bash scripts/r2_round8.sh

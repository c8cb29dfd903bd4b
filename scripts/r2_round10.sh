#!/bin/bash
# LEAN 3 (material-0 tiles holding tets and hexes): parity subset, A/B on cfg5 against the previous library
out=gpurun_out/r10; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_extensions.py tests/test_gpu_robustness.py tests/test_gpu_dist.py tests/test_gpu_dist_host.py -m gpu -x -q > $out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -5 $out/pytest_quick.log
sw() { timeout 600 python scripts/sweep.py --modes -1 --stages 2 --steps 100 --bench-layout "$@" 2>&1 | grep "part_nodes\|Error\|error" ; }
PREV=$PWD/paper_1909_05098_b200/libfedheat_b200_prev.so
for rep in 1 2; do
  for lib in prev new; do
    if [ $lib = prev ]; then L=$PREV; else L=""; fi
    for c in "cfg5 32" "cfg4 32"; do set -- $c; FH_LIB=$L sw --config $1 --precision $2 --parts 0 --check | sed "s/^/$lib $1 f$2 rep$rep /"; done
  done
done | tee $out/ab.jsonl
python - <<'PY' | tee $out/layout_cfg5.txt
import bench, paper_1909_05098_b200 as fh
prob = bench.make_problem("cfg5", 0, 32)
eng = fh.ExplicitEngine(prob.mesh, prob.material, prob.boundary, assembly="tiled", n_domains=8, **prob.engine_kwargs())
print({k: v for k, v in eng.layout().items() if k in ("kernels_per_step", "n_parts", "n_slots")})
PY

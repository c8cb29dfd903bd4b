#!/bin/bash
# T-only staging (two-knot laws): quick parity, then same-box A/B against the
# previous library (libfedheat_b200_old.so) and a tile-size sweep.
out=gpurun_out/tonly; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_extensions.py tests/test_gpu_resident.py -m gpu -x -q > $out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_quick.log
OLD=$PWD/paper_1909_05098_b200/libfedheat_b200_old.so
for rep in 1 2; do
  for lib in old new mb5; do
    if [ $lib = old ]; then L=$OLD; elif [ $lib = mb5 ]; then L=$PWD/paper_1909_05098_b200/libfedheat_b200_mb5.so; else L=""; fi
    for c in "cfg4 32" "cfg3 32" "cfg3 64" "cfg5 32"; do
      set -- $c
      FH_LIB=$L timeout 400 python scripts/sweep.py --config $1 --precision $2 --parts 0 --modes -1 --stages 2 --steps 100 --bench-layout 2>&1 | grep part_nodes | sed "s/^/$lib $1 f$2 rep$rep /"
    done
  done
done | tee $out/ab.jsonl
FH_LIB=$PWD/paper_1909_05098_b200/libfedheat_b200_mb5.so timeout 600 python scripts/sweep.py --config cfg4 --parts 1280,1408,1536,1664 --modes -1 --stages 2 --steps 100 --bench-layout 2>&1 | grep part_nodes | sed "s/^/sweep-mb5 cfg4 /" | tee $out/sweep_cfg4_mb5.jsonl
timeout 600 python scripts/sweep.py --config cfg4 --parts 1536,1792,2048,2304 --modes -1 --stages 2 --steps 100 --bench-layout 2>&1 | grep part_nodes | sed "s/^/sweep cfg4 /" | tee $out/sweep_cfg4.jsonl
timeout 600 python scripts/sweep.py --config cfg3 --precision 32 --parts 640,768,896,1024,1280 --modes -1 --stages 2 --steps 100 --bench-layout 2>&1 | grep part_nodes | sed "s/^/sweep cfg3 f32 /" | tee $out/sweep_cfg3_f32.jsonl
timeout 600 python scripts/sweep.py --config cfg3 --precision 64 --parts 512,640,768,896,1024 --modes -1 --stages 2 --steps 100 --bench-layout 2>&1 | grep part_nodes | sed "s/^/sweep cfg3 f64 /" | tee $out/sweep_cfg3_f64.jsonl

#!/bin/bash
# Round-end evidence on one GPU (part 1: small outputs): full GPU test suite,
# smoke, every bench line, ncu launch list of the default bench.  The ncu
# --set full captures (15-25 MB each) go in separate calls:
#   scripts/profile_cfg.sh cfg4 cfg3 ; scripts/profile_cfg.sh cfg5
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/final/smi.txt
rm -f gpurun_out/final/parity_fullsize.jsonl
FH_PARITY_JSON=$PWD/gpurun_out/final/parity_fullsize.jsonl timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
bash scripts/bench_all.sh
mkdir -p gpurun_out/prof
cmd="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/prof/launches.csv $cmd > gpurun_out/prof/ncu_launches.log 2>&1; echo "launches rc=$?"

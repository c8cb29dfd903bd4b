#!/bin/bash
# Round-end evidence on one GPU: full GPU test suite, smoke, every bench line,
# ncu launch list of the default bench and full captures of the step kernel.
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/final/smi.txt
timeout 1200 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
bash scripts/bench_all.sh
bash scripts/profile_round.sh
bash scripts/profile_cfg.sh cfg5

#!/bin/bash
# Round-2 state check on one GPU: full GPU suite + default bench line.
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 -p no:cacheprovider > gpurun_out/r2a/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2a/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/r2a/cfg4.json 2> gpurun_out/r2a/cfg4.err; echo "bench rc=$?"

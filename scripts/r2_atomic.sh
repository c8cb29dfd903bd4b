#!/bin/bash
mkdir -p gpurun_out/r2f
timeout 900 python -m pytest tests/test_gpu_atomic.py -q -x -p no:cacheprovider > gpurun_out/r2f/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2f/pytest.log
timeout 900 python scripts/atomic_vs_tiled.py cfg4 cfg3 > gpurun_out/r2f/ab.log 2>&1; echo "ab rc=$?"

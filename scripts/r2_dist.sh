#!/bin/bash
mkdir -p gpurun_out/r2e
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_fullsize.py --ignore=tests/reference_suite -k "not fullsize" > gpurun_out/r2e/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2e/pytest.log

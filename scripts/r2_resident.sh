#!/bin/bash
mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py tests/test_gpu_extensions.py tests/test_gpu_robustness.py tests/test_gpu_acceptance.py tests/test_gpu_solver_api.py tests/test_gpu_outputs.py -q -x -p no:cacheprovider > gpurun_out/r2b/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2b/pytest.log
timeout 300 python scripts/resident_sweep.py cfg1 1000 > gpurun_out/r2b/sweep_cfg1.log 2>&1; echo "sweep1 rc=$?"
timeout 300 python scripts/resident_sweep.py cfg2 2000 > gpurun_out/r2b/sweep_cfg2.log 2>&1; echo "sweep2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o gpurun_out/r2b/resident_cfg1 python scripts/resident_sweep.py cfg1 200 > gpurun_out/r2b/ncu.log 2>&1; echo "ncu rc=$?"

#!/bin/bash
# stamped-word synchronisation of the resident kernel: tests, then the sweep against the grid barrier
out=gpurun_out/stamped; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_races.py tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_solver_api.py -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
timeout 300 python scripts/resident_sweep.py cfg1 1000 > $out/sweep_cfg1.log 2>&1; echo "sweep1 rc=$?"; cat $out/sweep_cfg1.log
timeout 300 python scripts/resident_sweep.py cfg2 2000 > $out/sweep_cfg2.log 2>&1; echo "sweep2 rc=$?"; cat $out/sweep_cfg2.log

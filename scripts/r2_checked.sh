#!/bin/bash
# the GPU suite (full-size oracle runs excluded) on the bounds-checked build,
# then the schedule-invariance tests on the production build
mkdir -p gpurun_out/r2g
FH_LIB=$PWD/paper_1909_05098_b200/libfedheat_b200_checked.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/reference_suite --deselect tests/test_gpu_fullsize.py -k "not fullsize and not full_size" > gpurun_out/r2g/pytest_checked.log 2>&1; echo "checked rc=$?"; tail -3 gpurun_out/r2g/pytest_checked.log
timeout 900 python -m pytest tests/test_gpu_races.py -q -p no:cacheprovider > gpurun_out/r2g/races.log 2>&1; echo "races rc=$?"; tail -3 gpurun_out/r2g/races.log

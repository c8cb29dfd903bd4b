#!/bin/bash
# repeat the synchronisation-sensitive GPU tests (stamped resident kernel, TMA ring, host-transport processes)
out=gpurun_out/flake; mkdir -p $out
fails=0
for k in $(seq 1 ${1:-15}); do
  timeout 600 python -m pytest tests/test_gpu_resident.py tests/test_gpu_races.py tests/test_gpu_parity.py tests/test_gpu_robustness.py -m gpu -q -x -p no:cacheprovider > $out/run_$k.log 2>&1 || { fails=$((fails+1)); echo "run $k FAILED"; tail -5 $out/run_$k.log; }
done
echo "repeat runs: ${1:-15}, failures: $fails" | tee $out/summary.txt
tail -1 $out/run_1.log >> $out/summary.txt

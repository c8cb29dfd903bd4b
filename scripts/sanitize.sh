#!/bin/bash
# compute-sanitizer evidence for the step kernels (small meshes)
out=gpurun_out/san; mkdir -p $out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --log-file $out/$tool.log python scripts/sanitize_driver.py > $out/$tool.out 2>&1
  echo "$tool rc=$?"; tail -2 $out/$tool.log
done

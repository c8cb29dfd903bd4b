#!/bin/bash
# quick bench lines: OUT dir, configs as "name:args" words
out=${OUT:-gpurun_out/qb}; mkdir -p $out
for spec in "$@"; do
  name=${spec%%:*}; a=${spec#*:}; a=${a//,/ }
  timeout 600 python bench.py $a > $out/$name.json 2> $out/$name.err; echo "$name rc=$?"
done

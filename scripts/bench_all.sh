#!/bin/bash
# Run bench.py on every workload (one GPU) and keep the JSON lines.
out=${OUT:-gpurun_out/bench}
mkdir -p $out
python bench.py > $out/cfg4.json 2> $out/cfg4.err; echo "cfg4 rc=$?"
python bench.py --impl reference > $out/ref_cfg4.json 2> $out/ref_cfg4.err; echo "ref rc=$?"
python bench.py --config cfg1 --steps 1000 > $out/cfg1.json 2> $out/cfg1.err; echo "cfg1 rc=$?"
python bench.py --config cfg2 --steps 2000 > $out/cfg2_f64.json 2> $out/cfg2_f64.err; echo "cfg2 f64 rc=$?"
python bench.py --config cfg2 --steps 2000 --precision 32 --no-cpu-baseline > $out/cfg2_f32.json 2> $out/cfg2_f32.err; echo "cfg2 f32 rc=$?"
python bench.py --config cfg3 --precision 32 > $out/cfg3_f32.json 2> $out/cfg3_f32.err; echo "cfg3 f32 rc=$?"
python bench.py --config cfg3 --precision 64 --no-cpu-baseline > $out/cfg3_f64.json 2> $out/cfg3_f64.err; echo "cfg3 f64 rc=$?"
python bench.py --config cfg5 --steps 100 > $out/cfg5.json 2> $out/cfg5.err; echo "cfg5 rc=$?"

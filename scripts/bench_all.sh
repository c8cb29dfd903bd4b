#!/bin/bash
# Run bench.py on every workload (one GPU) and keep the JSON lines.
mkdir -p gpurun_out/bench
python bench.py > gpurun_out/bench/cfg4.json 2> gpurun_out/bench/cfg4.err; echo "cfg4 rc=$?"
python bench.py --config cfg3 --precision 32 > gpurun_out/bench/cfg3_f32.json 2> gpurun_out/bench/cfg3_f32.err; echo "cfg3 f32 rc=$?"
python bench.py --config cfg3 --precision 64 --no-cpu-baseline > gpurun_out/bench/cfg3_f64.json 2> gpurun_out/bench/cfg3_f64.err; echo "cfg3 f64 rc=$?"
python bench.py --config cfg5 --steps 100 > gpurun_out/bench/cfg5.json 2> gpurun_out/bench/cfg5.err; echo "cfg5 rc=$?"
python bench.py --config cfg1 --steps 1000 > gpurun_out/bench/cfg1.json 2> gpurun_out/bench/cfg1.err; echo "cfg1 rc=$?"
python bench.py --config cfg2 --steps 2000 --precision 32 --no-cpu-baseline > gpurun_out/bench/cfg2_f32.json 2> gpurun_out/bench/cfg2_f32.err; echo "cfg2 rc=$?"
python bench.py --impl reference > gpurun_out/bench/ref_cfg4.json 2> gpurun_out/bench/ref_cfg4.err; echo "ref rc=$?"

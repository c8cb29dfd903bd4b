#!/bin/bash
# ncu --set full captures of the step kernels (one step each), summarised ON THE BOX
# (the reports together exceed gpurun's 64 MiB return limit; only cfg4's comes back)
out=gpurun_out/prof2; rm -rf $out; mkdir -p $out
rm -rf gpurun_out/prof gpurun_out/tonly gpurun_out/r3 gpurun_out/r4 gpurun_out/r5
summ() {  # summ CONFIG PRECISION
  rep=$out/tiled_$1_f$2.ncu-rep
  { echo "# ncu --set full --clock-control none --import-source on, k_tiled_step launch(es) of one step of bench.py --config $1 --precision $2 --steps 20 --warmup 3 (round 2, T-only staging, 5/6 CTAs per SM)"
    python scripts/ncu_summary.py $rep
    echo; echo "# hottest basic blocks (scripts/ncu_stalls.py)"
    python scripts/ncu_stalls.py $rep; } > $out/r2b_ncu_tiled_$1_f$2.txt 2>&1
}
bash scripts/r2_prof.sh cfg4 32 1; summ cfg4 32
bash scripts/r2_prof.sh cfg3 32 1; summ cfg3 32; rm -f $out/tiled_cfg3_f32.ncu-rep
bash scripts/r2_prof.sh cfg3 64 1; summ cfg3 64; rm -f $out/tiled_cfg3_f64.ncu-rep
bash scripts/r2_prof.sh cfg5 32 3; summ cfg5 32; rm -f $out/tiled_cfg5_f32.ncu-rep
for c in cfg4 cfg5 cfg1; do
  cmd="python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $out/launches_$c.csv $cmd > $out/ncu_launches_$c.log 2>&1; echo "launches $c rc=$?"
done
ls -la $out; du -sh gpurun_out

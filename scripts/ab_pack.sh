mkdir -p gpurun_out/ab2
for rep in 1 2; do
for v in 1 0; do
  for c in cfg3 cfg5; do
    FH_NPH_PACK=$v timeout 300 python bench.py --config $c --steps 100 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab2/$c.$v.json 2>/dev/null
    echo "pack=$v $c $(python -c "import json;d=json.loads(open('gpurun_out/ab2/$c.$v.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4))")"
  done
done
done

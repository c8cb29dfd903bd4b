#!/bin/bash
# e2e (host buffers, double-buffered) repeatability on one box
mkdir -p gpurun_out/e2e
for r in 1 2 3; do
  for c in cfg4 cfg5; do
    timeout 400 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-steps 40 > gpurun_out/e2e/$c.$r.json 2>/dev/null
    echo "$c run $r e2e $(python -c "import json;d=json.loads(open('gpurun_out/e2e/$c.$r.json').read().strip().splitlines()[-1]);e=d['e2e'];print('%.3g'%e['value'], round((e['h2d_bytes_per_step']+e['d2h_bytes_per_step'])/(d['config']['elements']/e['value'])/1e9,1),'GB/s')")"
  done
done
